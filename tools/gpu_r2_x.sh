#!/bin/bash
# round-2 X: GroupNorm kernels -- launch list of one 1024^2 step (time + DRAM bytes), ncu --set full of
# the largest concat-input statistics pass and one apply; isolated GN timings
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/x_build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/x_launches_n1.csv python tools/prof_step.py 1 128 sdxl 1 > gpurun_out/x_prof_n1.out 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gn_stats -s 8 -c 1 -o gpurun_out/x_full_gn_stats python tools/prof_step.py 1 128 sdxl 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gn_apply -s 2 -c 1 -o gpurun_out/x_full_gn_apply python tools/prof_step.py 1 128 sdxl 1 > /dev/null 2>&1
timeout 300 python tools/bench_ops.py > gpurun_out/x_bench_ops.txt 2>&1
ls -la gpurun_out | grep x_
