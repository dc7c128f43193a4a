# round-1 evidence: bench line, per-op device times, ncu launch list (+DRAM bytes), ncu --set full captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/r1_bench_n1.json 2> gpurun_out/r1_bench_n1.err; tail -1 gpurun_out/r1_bench_n1.json
PCPP_OP_TIMING=1 timeout 200 python bench.py --no-cpu --no-e2e --steps 3 2> gpurun_out/r1_optiming.err > /dev/null; grep -E "^op" gpurun_out/r1_optiming.err > gpurun_out/r1_optiming.txt
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 9000 --csv --log-file gpurun_out/r1_launches_v3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile > /dev/null 2>&1
for spec in "gemm_tc_kernel:3" "attn_tc_kernel:0" "attn_tc_kernel:4" "gn_apply_wide:0" "gn_finalize:0"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/r1_full_${k}_$s python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile > /dev/null 2>&1
done
ls -la gpurun_out
