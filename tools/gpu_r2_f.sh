#!/bin/bash
# round-2 F: in-kernel GN finalize; full GPU suite; bench N = 2 code path on one GPU (PEER, gloo)
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/f_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/f_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/f_gpu.log
PCPP_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/f_bench2.json 2> gpurun_out/f_bench2.err; echo "bench2 rc=$?" >> gpurun_out/f_bench2.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?" >> gpurun_out/f_bench.err
timeout 300 python tools/optiming_n.py 1 > gpurun_out/f_opt_n1.txt 2>&1
tail -n 5 gpurun_out/f_gpu.log; tail -n 3 gpurun_out/f_bench2.err gpurun_out/f_bench.err
