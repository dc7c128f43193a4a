timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py tests/test_gpu_path.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do timeout 200 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench_f.log 2>&1; echo "rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bench_f.log').read().strip().splitlines()[-1]);print(d['value'],d['breakdown_ms'])"; done
