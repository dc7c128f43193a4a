#!/bin/bash
# round-2 J: stream-K attention -- op / full-size / path / golden parity, graph-timed scaling, bench
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/j_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py -q -x > gpurun_out/j_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/j_ops.log
timeout 600 python tools/graph_timing.py attn-scaling > gpurun_out/j_attn.txt 2>&1
PCPP_GEMM_FORCE=160,1,0 timeout 300 python tools/gemm_trace.py > gpurun_out/j_trace160.txt 2>&1
PCPP_GEMM_FORCE=160,1,0 timeout 300 python tools/graph_timing.py gemm-scaling > gpurun_out/j_gemm.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf > gpurun_out/j_bench.json 2> gpurun_out/j_bench.err; echo "bench rc=$?" >> gpurun_out/j_bench.err
timeout 1200 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_xf.py tests/test_gpu_peer.py -q -x > gpurun_out/j_path.log 2>&1; echo "path rc=$?" >> gpurun_out/j_path.log
tail -n 3 gpurun_out/j_ops.log gpurun_out/j_path.log gpurun_out/j_bench.err; cat gpurun_out/j_attn.txt
