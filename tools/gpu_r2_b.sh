#!/bin/bash
# round-2 check B: xf models, PEER backend (deterministic configs), GN stats v2 (ops + golden), bench
cd $GRAFT_REPO_ROOT
free -g > gpurun_out/b_host.txt; nproc >> gpurun_out/b_host.txt
python paper_2412_02962_b200/build.py > gpurun_out/b_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_peer.py -q -s > gpurun_out/b_peer.log 2>&1; echo "peer rc=$?" >> gpurun_out/b_peer.log
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_golden.py -q > gpurun_out/b_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/b_ops.log
timeout 1200 python -m pytest tests/test_gpu_xf.py -q -s > gpurun_out/b_xf.log 2>&1; echo "xf rc=$?" >> gpurun_out/b_xf.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-loopback > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; echo "bench rc=$?" >> gpurun_out/b_bench.err
for f in gpurun_out/b_peer.log gpurun_out/b_ops.log gpurun_out/b_xf.log gpurun_out/b_bench.err; do tail -n 4 $f; done
