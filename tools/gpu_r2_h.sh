#!/bin/bash
# round-2 H: GEMM launch timeline (globaltimer stamps); revert of the in-kernel finalize (bench)
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/h_build.log 2>&1
PCPP_GEMM_FORCE=160,1,0 timeout 300 python tools/gemm_trace.py > gpurun_out/h_trace160.txt 2>&1
PCPP_GEMM_FORCE=64,1,0 timeout 300 python tools/gemm_trace.py > gpurun_out/h_trace64.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo "bench rc=$?" >> gpurun_out/h_bench.err
cat gpurun_out/h_trace160.txt; tail -n 2 gpurun_out/h_bench.err
