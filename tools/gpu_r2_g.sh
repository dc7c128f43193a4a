#!/bin/bash
# round-2 G: in-kernel GN finalize v2 (parallel slot reduction); attention / GEMM scaling (graph-timed)
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/g_build.log 2>&1
timeout 600 python tools/graph_timing.py attn-scaling > gpurun_out/g_attn.txt 2>&1
timeout 600 python tools/graph_timing.py gemm-scaling > gpurun_out/g_gemm.txt 2>&1
for f in "160,1,0" "64,1,0" "128,2,0" "256,1,1" "160,2,0"; do echo "FORCE $f" >> gpurun_out/g_gemm_force.txt; PCPP_GEMM_FORCE=$f timeout 300 python tools/graph_timing.py gemm-scaling >> gpurun_out/g_gemm_force.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py -q -x > gpurun_out/g_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo "bench rc=$?" >> gpurun_out/g_bench.err
cat gpurun_out/g_attn.txt; tail -n 3 gpurun_out/g_tests.log gpurun_out/g_bench.err
