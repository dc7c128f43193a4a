timeout 900 python -m pytest tests/test_gpu_path.py -m gpu -q -x -k forced 2>&1 | tail -3
PCPP_GEMM_LOG=1 timeout 200 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench_d.log 2>&1; echo rc=$?
grep gemm-tune gpurun_out/bench_d.log
python -c "import json;d=json.loads(open('gpurun_out/bench_d.log').read().strip().splitlines()[-1]);print(d['value'],d['breakdown_ms'])"
