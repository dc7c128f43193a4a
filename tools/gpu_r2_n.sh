#!/bin/bash
# round-2 N: attention O through smem + TMA store; GN stats with 8 loads in flight; tests + timing + bench
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/n_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py -q > gpurun_out/n_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/n_ops.log
timeout 600 python tools/graph_timing.py attn-scaling > gpurun_out/n_attn.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err; echo "bench rc=$?" >> gpurun_out/n_bench.err
timeout 300 python tools/optiming_n.py 1 > gpurun_out/n_opt_n1.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_xf.py tests/test_gpu_peer.py -q > gpurun_out/n_path.log 2>&1; echo "path rc=$?" >> gpurun_out/n_path.log
tail -n 3 gpurun_out/n_ops.log gpurun_out/n_path.log gpurun_out/n_bench.err; tail -n 4 gpurun_out/n_attn.txt
