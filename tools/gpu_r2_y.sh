#!/bin/bash
# round-2 Y: GroupNorm statistics + apply through TMA bulk-copy rings -- ops tests, GN op timings,
# same-box A/B against the register-load kernels (the tree minus gpurun_out/gn_bulk.patch), path tests
cd $GRAFT_REPO_ROOT
B="--steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e"
build() { python paper_2412_02962_b200/build.py > /dev/null 2>&1 || echo BUILD FAILED; }
run() { timeout 600 python bench.py $B 2>/dev/null | tail -1 > gpurun_out/y_$1.json; python -c "import json;d=json.load(open('gpurun_out/y_$1.json'));print('$1', d['value'],d['breakdown_ms'])"; }
build
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x > gpurun_out/y_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/y_ops.log
tail -2 gpurun_out/y_ops.log
timeout 300 python tools/bench_ops.py 2>&1 | grep GN > gpurun_out/y_gn_new.txt
run B1
patch -R -p1 < gpurun_out/gn_bulk.patch > /dev/null; build
timeout 300 python tools/bench_ops.py 2>&1 | grep GN > gpurun_out/y_gn_old.txt
run A1
patch -p1 < gpurun_out/gn_bulk.patch > /dev/null; build
run B2
patch -R -p1 < gpurun_out/gn_bulk.patch > /dev/null; build
run A2
patch -p1 < gpurun_out/gn_bulk.patch > /dev/null; build
cat gpurun_out/y_gn_old.txt gpurun_out/y_gn_new.txt
timeout 2400 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_peer.py tests/test_gpu_xf.py -q -x > gpurun_out/y_path.log 2>&1; echo "path rc=$?" >> gpurun_out/y_path.log
tail -n 3 gpurun_out/y_path.log
