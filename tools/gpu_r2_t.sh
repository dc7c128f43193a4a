#!/bin/bash
# round-2 T: 8 epilogue warps in the tcgen05 GEMMs (2 per TMEM lane quadrant) -- bench with the committed
# table, a fresh autotune table over every bench shape, bench with it, trace, tests
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/t_build.log 2>&1
B="--steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e"
timeout 600 python bench.py $B > gpurun_out/t_bench_old.json 2> gpurun_out/t_bench_old.err; echo "bench rc=$?" >> gpurun_out/t_bench_old.err
PCPP_TUNE_FILE=/nonexistent PCPP_TUNE_SAVE=gpurun_out/t_tune.txt timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/t_bench_tune.json 2> gpurun_out/t_bench_tune.err; echo "tune rc=$?" >> gpurun_out/t_bench_tune.err
PCPP_TUNE_FILE=gpurun_out/t_tune.txt timeout 600 python bench.py $B > gpurun_out/t_bench_new.json 2> gpurun_out/t_bench_new.err; echo "bench rc=$?" >> gpurun_out/t_bench_new.err
EPI=bias timeout 200 python tools/gemm_trace.py > gpurun_out/t_trace.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x > gpurun_out/t_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/t_ops.log
timeout 900 python -m pytest tests/test_gpu_path.py -q -x -k "forced" > gpurun_out/t_forced.log 2>&1; echo "forced rc=$?" >> gpurun_out/t_forced.log
timeout 1500 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_xf.py -q -x > gpurun_out/t_path.log 2>&1; echo "path rc=$?" >> gpurun_out/t_path.log
for f in t_bench_old t_bench_new; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['value'],d['breakdown_ms'])"; done
tail -n 2 gpurun_out/t_bench_tune.err gpurun_out/t_ops.log gpurun_out/t_forced.log gpurun_out/t_path.log
