#!/bin/bash
# round-2 L: cluster split-K GEMM -- correctness (op-level forced, whole path forced), timing, bench
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/l_build.log 2>&1
for f in "160,1,0" "160,1,2" "128,1,4" "64,1,4" "160,1,4" "256,1,2"; do PCPP_GEMM_FORCE=$f timeout 120 python tools/check_gemm_force.py >> gpurun_out/l_check.txt 2>&1; done
for f in "160,1,2" "160,1,4" "128,1,4" "64,1,4"; do echo "FORCE $f" >> gpurun_out/l_force.txt; PCPP_GEMM_FORCE=$f timeout 300 python tools/graph_timing.py gemm-scaling >> gpurun_out/l_force.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_path.py -q -k "forced" > gpurun_out/l_forced.log 2>&1; echo "forced rc=$?" >> gpurun_out/l_forced.log
PCPP_GEMM_LOG=1 timeout 300 python tools/optiming_n.py 8 > gpurun_out/l_opt_n8.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-large --no-xf > gpurun_out/l_bench.json 2> gpurun_out/l_bench.err; echo "bench rc=$?" >> gpurun_out/l_bench.err
grep -h "FORCE\|FAIL" gpurun_out/l_check.txt; tail -n 3 gpurun_out/l_forced.log gpurun_out/l_bench.err
