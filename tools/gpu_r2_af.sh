#!/bin/bash
# round-2 AF: conv_out with 12 warps per CTA (one kernel row per warp group, partials reduced in smem)
# -- same-box A/B (A = minus ab/cout12.patch), ncu of conv_out, path tests
cd $GRAFT_REPO_ROOT
B="--steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e"
build() { python paper_2412_02962_b200/build.py > /dev/null 2>&1 || echo BUILD FAILED; }
run() { timeout 600 python bench.py $B 2>/dev/null | tail -1 > gpurun_out/af_$1.json; python -c "import json;d=json.load(open('gpurun_out/af_$1.json'));print('$1', d['value'],d['breakdown_ms'])"; }
build
run N1
patch -R -p1 < ab/cout12.patch > /dev/null; build; run A1
patch -p1 < ab/cout12.patch > /dev/null; build; run N2
patch -R -p1 < ab/cout12.patch > /dev/null; build; run A2
patch -p1 < ab/cout12.patch > /dev/null; build
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_out -c 1 -o gpurun_out/af_full_conv_out python tools/prof_step.py 1 128 sdxl 1 > /dev/null 2>&1
timeout 2400 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py -q -x > gpurun_out/af_path.log 2>&1; echo "path rc=$?" >> gpurun_out/af_path.log
tail -n 2 gpurun_out/af_path.log
