#!/bin/bash
# round-2 D: cfg_split fix, per-op timing tables n = 1 / 8, launch lists with DRAM bytes
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/d_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_path.py -q -k "cfg_split" > gpurun_out/d_split.log 2>&1; echo "split rc=$?" >> gpurun_out/d_split.log
timeout 300 python tools/optiming_n.py 1 > gpurun_out/d_opt_n1.txt 2>&1
timeout 300 python tools/optiming_n.py 8 > gpurun_out/d_opt_n8.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/d_launches_n1.csv python tools/prof_step.py 1 128 sdxl 1 > gpurun_out/d_prof_n1.out 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/d_launches_n8.csv python tools/prof_step.py 8 128 sdxl 1 > gpurun_out/d_prof_n8.out 2>&1
tail -n 3 gpurun_out/d_split.log; tail -n 2 gpurun_out/d_opt_n1.txt gpurun_out/d_opt_n8.txt; ls -la gpurun_out/
