#!/bin/bash
# round-2 re-entry check: full GPU suite, smoke, default bench
cd $GRAFT_REPO_ROOT
nproc > gpurun_out/c_host.txt; lscpu | grep 'Model name' >> gpurun_out/c_host.txt; nvidia-smi -L >> gpurun_out/c_host.txt
python paper_2412_02962_b200/build.py > gpurun_out/c_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/c_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/c_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/c_smoke.log
timeout 900 python bench.py > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err; echo "bench rc=$?" >> gpurun_out/c_bench.err
tail -n 30 gpurun_out/c_gpu.log; tail -3 gpurun_out/c_smoke.log; tail -5 gpurun_out/c_bench.err
