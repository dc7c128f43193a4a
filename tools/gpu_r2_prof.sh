#!/bin/bash
# round-2 profiles: launch list of one 1024^2 step (time + DRAM bytes per launch), ncu --set full of
# the GroupNorm and attention kernels
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_n1.csv python tools/prof_step.py 1 128 sdxl 1 > gpurun_out/r2_prof_n1.out 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_n8.csv python tools/prof_step.py 8 128 sdxl 1 > gpurun_out/r2_prof_n8.out 2>&1
for spec in "gn_apply_wide:10" "gn_stats_kernel:3" "attn_tc_kernel:30" "gn_finalize:10"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/r2_full_${k} python tools/prof_step.py 1 128 sdxl 1 > /dev/null 2>&1
done
ls -la gpurun_out | grep r2_
