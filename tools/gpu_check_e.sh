timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for v in 1 0 1; do PCPP_GN_WIDE=$v timeout 200 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench_e.log 2>&1; echo "wide=$v rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bench_e.log').read().strip().splitlines()[-1]);print(d['value'],d['breakdown_ms'])"; done
