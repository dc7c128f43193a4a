# round-1 final evidence (run on one B200): tests, smoke, bench (both arms), ncu launch list + full captures
set -x
python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/r1_bench_n1.json 2> gpurun_out/r1_bench_n1.err; tail -c 600 gpurun_out/r1_bench_n1.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1_bench_reference_n1.json 2>/dev/null; tail -c 300 gpurun_out/r1_bench_reference_n1.json
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 9000 --csv --log-file gpurun_out/r1_launches_v4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile --no-loopback > /dev/null 2>&1
for spec in "gemm_tc_kernel:3" "gemm_tc2_kernel:3" "attn_tc_kernel:0" "attn_tc_kernel:4" "gn_apply_wide:0"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/r1f_${k}_$s python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile --no-loopback > /dev/null 2>&1
done
ls -la gpurun_out | grep r1
