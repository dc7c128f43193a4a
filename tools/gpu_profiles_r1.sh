# round-1 evidence: ncu launch list (+DRAM bytes) of one step, ncu --set full captures of the top kernels
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 9000 --csv --log-file gpurun_out/r1_launches_v3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile > /dev/null 2>&1
for spec in "gemm_tc2_kernel:3" "gemm_tc_kernel:3" "attn_tc_kernel:0" "attn_tc_kernel:4" "gn_apply_wide:0"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/r1_full_${k}_$s python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile > /dev/null 2>&1
done
ls -la gpurun_out | grep r1_
