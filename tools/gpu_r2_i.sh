#!/bin/bash
# round-2 I: staged TMA-store GEMM epilogue -- correctness (ops, path, golden), A/B timing, bench
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/i_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_path.py -q -x > gpurun_out/i_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/i_tests.log
for st in 1 0; do echo "TMA_STORE=$st" >> gpurun_out/i_ab.txt; PCPP_GEMM_TMA_STORE=$st PCPP_GEMM_FORCE=160,1,0 timeout 300 python tools/graph_timing.py gemm-scaling >> gpurun_out/i_ab.txt 2>&1; done
PCPP_GEMM_FORCE=160,1,0 timeout 300 python tools/gemm_trace.py > gpurun_out/i_trace160.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err; echo "bench rc=$?" >> gpurun_out/i_bench.err
PCPP_GEMM_TMA_STORE=0 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback > gpurun_out/i_bench_off.json 2> gpurun_out/i_bench_off.err
timeout 900 python -m pytest tests/test_gpu_golden.py -q -x > gpurun_out/i_golden.log 2>&1; echo "golden rc=$?" >> gpurun_out/i_golden.log
tail -n 3 gpurun_out/i_tests.log gpurun_out/i_golden.log gpurun_out/i_bench.err; cat gpurun_out/i_ab.txt
