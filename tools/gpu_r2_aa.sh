#!/bin/bash
# round-2 AA: (D) kernels end on read-completion of their bulk / TMA stores (not write completion) +
# GN apply sums all producer slots (no finalize); vs (B) write-completion waits; then a fresh autotune
# table with the best-of-2-trials tuner (E) against the committed table
cd $GRAFT_REPO_ROOT
B="--steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e"
build() { python paper_2412_02962_b200/build.py > /dev/null 2>&1 || echo BUILD FAILED; }
run() { timeout 600 python bench.py $B 2>/dev/null | tail -1 > gpurun_out/aa_$1.json; python -c "import json;d=json.load(open('gpurun_out/aa_$1.json'));print('$1', d['value'],d['breakdown_ms'])"; }
build
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x > gpurun_out/aa_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/aa_ops.log
tail -1 gpurun_out/aa_ops.log
run D1
patch -R -p1 < ab/readwait.patch > /dev/null; build; run B1
patch -p1 < ab/readwait.patch > /dev/null; build; run D2
patch -R -p1 < ab/readwait.patch > /dev/null; build; run B2
patch -p1 < ab/readwait.patch > /dev/null; build
PCPP_TUNE_FILE=/nonexistent PCPP_TUNE_SAVE=gpurun_out/aa_tune.txt timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/aa_tune_bench.json 2> gpurun_out/aa_tune_bench.err; echo "tune rc=$?"
for i in 1 2; do PCPP_TUNE_FILE=gpurun_out/aa_tune.txt timeout 600 python bench.py $B 2>/dev/null | tail -1 > gpurun_out/aa_E$i.json; python -c "import json;d=json.load(open('gpurun_out/aa_E$i.json'));print('E$i', d['value'],d['breakdown_ms'])"; run D$((i+2)); done
timeout 2400 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_peer.py tests/test_gpu_xf.py -q -x > gpurun_out/aa_path.log 2>&1; echo "path rc=$?" >> gpurun_out/aa_path.log
tail -n 2 gpurun_out/aa_path.log
