#!/bin/bash
# round-2 AC: (T) attention splits a short last wave's units over up to 4 CTAs (last-arriver combine)
# + conv_out on warp-level tensor-core MMAs (hi/lo bf16 weights); same-box A/B of the attention split
# (A = minus ab/tailsplit.patch), attention graph timings, ncu of conv_out, tests
cd $GRAFT_REPO_ROOT
B="--steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e"
build() { python paper_2412_02962_b200/build.py > /dev/null 2>&1 || echo BUILD FAILED; }
run() { timeout 600 python bench.py $B 2>/dev/null | tail -1 > gpurun_out/ac_$1.json; python -c "import json;d=json.load(open('gpurun_out/ac_$1.json'));print('$1', d['value'],d['breakdown_ms'])"; }
build
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x > gpurun_out/ac_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/ac_ops.log; tail -1 gpurun_out/ac_ops.log
run T1
patch -R -p1 < ab/tailsplit.patch > /dev/null; build; run A1
patch -p1 < ab/tailsplit.patch > /dev/null; build; run T2
patch -R -p1 < ab/tailsplit.patch > /dev/null; build; run A2
patch -p1 < ab/tailsplit.patch > /dev/null; build
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_out -c 1 -o gpurun_out/ac_full_conv_out python tools/prof_step.py 1 128 sdxl 1 > /dev/null 2>&1
timeout 2400 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_peer.py tests/test_gpu_xf.py tests/test_gpu_fullsize.py -q -x > gpurun_out/ac_path.log 2>&1; echo "path rc=$?" >> gpurun_out/ac_path.log
tail -n 2 gpurun_out/ac_path.log
