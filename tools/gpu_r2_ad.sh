#!/bin/bash
# round-2 AD: bulk-copy GroupNorm apply for channel-concat inputs (separate double-buffered output
# stages) -- same-box A/B (A = minus ab/catapply.patch), GN op timings, path tests
cd $GRAFT_REPO_ROOT
B="--steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e"
build() { python paper_2412_02962_b200/build.py > /dev/null 2>&1 || echo BUILD FAILED; }
run() { timeout 600 python bench.py $B 2>/dev/null | tail -1 > gpurun_out/ad_$1.json; python -c "import json;d=json.load(open('gpurun_out/ad_$1.json'));print('$1', d['value'],d['breakdown_ms'])"; }
build
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x > gpurun_out/ad_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/ad_ops.log; tail -1 gpurun_out/ad_ops.log
run C1
patch -R -p1 < ab/catapply.patch > /dev/null; build; run A1
patch -p1 < ab/catapply.patch > /dev/null; build; run C2
patch -R -p1 < ab/catapply.patch > /dev/null; build; run A2
patch -p1 < ab/catapply.patch > /dev/null; build; run C3
timeout 2400 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_fullsize.py -q -x > gpurun_out/ad_path.log 2>&1; echo "path rc=$?" >> gpurun_out/ad_path.log
tail -n 2 gpurun_out/ad_path.log
