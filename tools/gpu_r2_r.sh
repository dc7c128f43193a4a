#!/bin/bash
# round-2 R: GN-fused GEMMs keep the full ring (register group accumulators, stats from the staging tile)
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/r_build.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err; echo "bench rc=$?" >> gpurun_out/r_bench.err
timeout 900 python -m pytest tests/test_gpu_path.py -q -k "forced" > gpurun_out/r_forced.log 2>&1; echo "forced rc=$?" >> gpurun_out/r_forced.log
timeout 1500 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_peer.py tests/test_gpu_xf.py tests/test_gpu_ops.py -q > gpurun_out/r_path.log 2>&1; echo "path rc=$?" >> gpurun_out/r_path.log
tail -n 3 gpurun_out/r_forced.log gpurun_out/r_path.log gpurun_out/r_bench.err
