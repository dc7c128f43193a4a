#!/bin/bash
# round-2 M: retune the GEMM table (all 1024^2 shapes, n = 1/2/4/8, incl. cluster split-K); launch lists of
# one step (n = 1, n = 8) with DRAM bytes; ncu --set full of the top kernels
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/m_build.log 2>&1
PCPP_TUNE_FILE=/nonexistent PCPP_TUNE_SAVE=gpurun_out/gemm_tune_b200.txt timeout 1500 python bench.py --steps 5 --warmup 3 --no-cpu --no-xf --no-large > gpurun_out/m_tune_bench.json 2> gpurun_out/m_tune_bench.err
export PCPP_TUNE_FILE=$GRAFT_REPO_ROOT/gpurun_out/gemm_tune_b200.txt
export PROF_RANGE=1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches_n1.csv python tools/prof_step.py 1 128 sdxl 1 > gpurun_out/m_prof_n1.out 2>&1
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches_n8.csv python tools/prof_step.py 8 128 sdxl 1 > gpurun_out/m_prof_n8.out 2>&1
for spec in "gemm_tc_kernel:3:l0conv" "gemm_tc_kernel:150:l2gemm" "attn_tc_kernel:40:attn_l2" "attn_tc_kernel:2:attn_l1" "gn_apply_wide:10:gn_apply" "gn_stats_kernel:2:gn_stats"; do
  k=$(echo $spec | cut -d: -f1); sk=$(echo $spec | cut -d: -f2); tag=$(echo $spec | cut -d: -f3)
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -s $sk -c 1 -o gpurun_out/r2_full_$tag python tools/prof_step.py 1 128 sdxl 1 > gpurun_out/m_full_$tag.out 2>&1
done
ls -la gpurun_out | grep -E "r2_|gemm_tune"; tail -n 2 gpurun_out/m_tune_bench.err
