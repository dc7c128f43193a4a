#!/bin/bash
# round-2 K: TMA-store epilogue fix (W = 48 tiles), bias / temb prefetch; ops + path + golden; pair-160 sweep; bench
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/k_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py -q > gpurun_out/k_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/k_ops.log
for f in "160,1,1" "128,1,1"; do echo "FORCE $f" >> gpurun_out/k_force.txt; PCPP_GEMM_FORCE=$f timeout 300 python tools/graph_timing.py gemm-scaling >> gpurun_out/k_force.txt 2>&1; done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf > gpurun_out/k_bench.json 2> gpurun_out/k_bench.err; echo "bench rc=$?" >> gpurun_out/k_bench.err
timeout 1500 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_xf.py tests/test_gpu_peer.py -q > gpurun_out/k_path.log 2>&1; echo "path rc=$?" >> gpurun_out/k_path.log
tail -n 3 gpurun_out/k_ops.log gpurun_out/k_path.log gpurun_out/k_bench.err
