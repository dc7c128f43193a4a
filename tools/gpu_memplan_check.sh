# memory plan: bench A/B (PCPP_MEMPLAN=0 vs default) + the full GPU suite with the plan on
run() { timeout 300 env $2 python bench.py --no-cpu --no-e2e --no-loopback --steps 10 2>/dev/null | tail -1 > gpurun_out/ab.json; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$1', d['value'],d['breakdown_ms'])"; }
run A PCPP_MEMPLAN=0; run B PCPP_MEMPLAN=1; run A PCPP_MEMPLAN=0; run B PCPP_MEMPLAN=1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=8 2>&1 | tail -14
