#!/bin/bash
# round-2 check A: PEER backend multi-process tests, golden parity, path tests, a short bench
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/a_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q -s > gpurun_out/a_peer.log 2>&1; echo "peer rc=$?" >> gpurun_out/a_peer.log
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_path.py -q -s > gpurun_out/a_path.log 2>&1; echo "path rc=$?" >> gpurun_out/a_path.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err; echo "bench rc=$?" >> gpurun_out/a_bench.err
tail -3 gpurun_out/a_peer.log gpurun_out/a_path.log gpurun_out/a_bench.err
