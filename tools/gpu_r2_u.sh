#!/bin/bash
# round-2 U: double-buffered epilogue staging tiles -- ops tests, forced configs, bench x2, trace
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/u_build.log 2>&1
B="--steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e"
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x > gpurun_out/u_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/u_ops.log
for i in 1 2; do timeout 600 python bench.py $B > gpurun_out/u_bench$i.json 2> gpurun_out/u_bench$i.err; done
EPI=bias timeout 200 python tools/gemm_trace.py > gpurun_out/u_trace.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_path.py -q -x -k "forced" > gpurun_out/u_forced.log 2>&1; echo "forced rc=$?" >> gpurun_out/u_forced.log
for f in u_bench1 u_bench2; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['value'],d['breakdown_ms'])"; done
tail -n 2 gpurun_out/u_ops.log gpurun_out/u_forced.log; grep -A2 shape gpurun_out/u_trace.txt | head -12
