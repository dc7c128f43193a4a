#!/bin/bash
# round-2 P: GN finalize merged into the apply for small slot counts; apply loads before its prologue
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/p_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ops.py -q > gpurun_out/p_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/p_ops.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err; echo "bench rc=$?" >> gpurun_out/p_bench.err
timeout 1500 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_peer.py tests/test_gpu_xf.py -q > gpurun_out/p_path.log 2>&1; echo "path rc=$?" >> gpurun_out/p_path.log
tail -n 3 gpurun_out/p_ops.log gpurun_out/p_path.log gpurun_out/p_bench.err
