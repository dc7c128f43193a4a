#!/bin/bash
# round-2 Q: coalesced residual through the staging tile, bias+temb combined (one shuffle), read-only
# end waits; GN slot-sum loads in flight -- epilogue trace, correctness, bench
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/q_build.log 2>&1
for e in none bias+temb bias+temb+res; do EPI=$e PCPP_GEMM_FORCE=160,1,0 timeout 200 python tools/gemm_trace.py 2>&1 | grep -A2 "shape rows=4 W=32 K=1280 N=1280 taps=1\|shape rows=32 W=32 K=1280 N=1280" >> gpurun_out/q_trace.txt; done
for f in "160,1,0" "160,1,2" "128,1,4" "256,1,1"; do PCPP_GEMM_FORCE=$f timeout 120 python tools/check_gemm_force.py >> gpurun_out/q_check.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_ops.py -q > gpurun_out/q_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/q_ops.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo "bench rc=$?" >> gpurun_out/q_bench.err
timeout 1800 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_peer.py tests/test_gpu_xf.py -q > gpurun_out/q_path.log 2>&1; echo "path rc=$?" >> gpurun_out/q_path.log
cat gpurun_out/q_trace.txt; grep -h "FORCE" gpurun_out/q_check.txt; tail -n 3 gpurun_out/q_ops.log gpurun_out/q_path.log gpurun_out/q_bench.err
