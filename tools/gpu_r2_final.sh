#!/bin/bash
# round-2 final evidence: the driver's GPU suite, smoke, default bench (N = 1), reference arm, the N = 2
# code path on one GPU, compute-sanitizer on the new kernels
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f2_build.log 2>&1
timeout 1800 python -m pytest tests/ -x -q -m gpu > gpurun_out/f2_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/f2_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f2_smoke.log
timeout 900 python bench.py > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; echo "bench rc=$?" >> gpurun_out/f2_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f2_bench_ref.json 2> gpurun_out/f2_bench_ref.err; echo "ref rc=$?" >> gpurun_out/f2_bench_ref.err
PCPP_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/f2_bench2.json 2> gpurun_out/f2_bench2.err; echo "bench2 rc=$?" >> gpurun_out/f2_bench2.err
timeout 1500 bash tools/gpu_sanitize.sh > gpurun_out/f2_sanitizer.txt 2>&1
tail -n 3 gpurun_out/f2_gpu.log gpurun_out/f2_smoke.log gpurun_out/f2_bench.err gpurun_out/f2_bench_ref.err gpurun_out/f2_bench2.err; grep -E "ERROR SUMMARY|==" gpurun_out/f2_sanitizer.txt | head -30
