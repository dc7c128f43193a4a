start=$(date +%s)
timeout 900 python bench.py > gpurun_out/r1_bench_n1.json 2> gpurun_out/r1_bench_n1.err
echo "bench wall s: $(( $(date +%s) - start ))"
tail -c 300 gpurun_out/r1_bench_n1.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1_bench_reference_n1.json 2>/dev/null
tail -c 200 gpurun_out/r1_bench_reference_n1.json
