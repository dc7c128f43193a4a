#!/bin/bash
# round-2 S (session 3): per-op device times of the 1024^2 step and the small-GEMM epilogue trace at HEAD
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/s_build.log 2>&1
PCPP_OP_TIMING=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e > gpurun_out/s_bench.json 2> gpurun_out/s_optiming.txt; echo "bench rc=$?" >> gpurun_out/s_optiming.txt
for e in bias bias+temb+res; do EPI=$e timeout 200 python tools/gemm_trace.py >> gpurun_out/s_trace.txt 2>&1; done
tail -n 3 gpurun_out/s_optiming.txt; cat gpurun_out/s_bench.json | head -c 600
