#!/bin/bash
# round-2 Z: (B) GroupNorm apply sums the producer's slots itself at n = 1 (no finalize launches),
# (C) + bulk apply with separate double-buffered output stages and concat inputs -- same-box A/B/C
cd $GRAFT_REPO_ROOT
B="--steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e"
build() { python paper_2412_02962_b200/build.py > /dev/null 2>&1 || echo BUILD FAILED; }
run() { timeout 600 python bench.py $B 2>/dev/null | tail -1 > gpurun_out/z_$1.json; python -c "import json;d=json.load(open('gpurun_out/z_$1.json'));print('$1', d['value'],d['breakdown_ms'])"; }
build
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x > gpurun_out/z_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/z_ops.log
tail -2 gpurun_out/z_ops.log
run C1
patch -R -p1 < ab/apply2.patch > /dev/null; build; run B1
patch -R -p1 < ab/merge.patch > /dev/null; build; run A1
patch -p1 < ab/merge.patch > /dev/null; build; run B2
patch -p1 < ab/apply2.patch > /dev/null; build; run C2
timeout 2400 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_peer.py tests/test_gpu_xf.py -q -x > gpurun_out/z_path.log 2>&1; echo "path rc=$?" >> gpurun_out/z_path.log
tail -n 3 gpurun_out/z_path.log
