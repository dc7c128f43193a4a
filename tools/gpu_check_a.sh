set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8
python bench.py 2>&1 | tail -1 > gpurun_out/bench_a.json
cat gpurun_out/bench_a.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_a.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile > /dev/null 2>&1
ls -la gpurun_out
