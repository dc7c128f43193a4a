#!/bin/bash
# round-2 AB: conv_in v2 (64-token CTAs, staged input rows, 8 independent accumulators) -- bench x2,
# path tests, ncu --set full of conv_in and conv_out
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/ab_build.log 2>&1
B="--steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e"
for i in 1 2; do timeout 600 python bench.py $B 2>/dev/null | tail -1 > gpurun_out/ab_$i.json; python -c "import json;d=json.load(open('gpurun_out/ab_$i.json'));print('ab$i', d['value'],d['breakdown_ms'])"; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_in_kernel -c 1 -o gpurun_out/ab_full_conv_in python tools/prof_step.py 1 128 sdxl 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_out_v3 -c 1 -o gpurun_out/ab_full_conv_out python tools/prof_step.py 1 128 sdxl 1 > /dev/null 2>&1
timeout 2400 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py -q -x > gpurun_out/ab_path.log 2>&1; echo "path rc=$?" >> gpurun_out/ab_path.log
tail -n 2 gpurun_out/ab_path.log
