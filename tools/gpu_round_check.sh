set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5
python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1.json
cat gpurun_out/bench_r1.json
python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_ref_r1.json
cat gpurun_out/bench_ref_r1.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile > /dev/null 2>&1
for k in "gemm_tc_kernel<256>" "gemm_tc_kernel<160>" "attn_tc_kernel" "gn_stats" "gn_apply"; do
  n=$(echo $k | tr -dc 'a-z0-9_')
  ncu --set full --import-source on --clock-control none -k regex:"$k" -s 2 -c 1 -o gpurun_out/prof_r1_$n python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile > /dev/null 2>&1
done
ls -la gpurun_out
