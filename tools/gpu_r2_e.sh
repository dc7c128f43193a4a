#!/bin/bash
# round-2 E: split-K for GN-fused GEMMs; X1 / SW goldens; per-op n = 8; bench (no extras)
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/e_build.log 2>&1
PCPP_GEMM_LOG=1 timeout 300 python tools/optiming_n.py 8 > gpurun_out/e_opt_n8.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_golden.py -q -s > gpurun_out/e_golden.log 2>&1; echo "golden rc=$?" >> gpurun_out/e_golden.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err; echo "bench rc=$?" >> gpurun_out/e_bench.err
tail -n 3 gpurun_out/e_golden.log gpurun_out/e_bench.err; tail -n 2 gpurun_out/e_opt_n8.txt
