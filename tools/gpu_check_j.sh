timeout 900 python -m pytest tests/test_gpu_path.py -m gpu -q -x -k "dpmpp or path_matches" 2>&1 | tail -3
timeout 200 python bench.py --no-cpu --no-e2e --steps 10 2>/dev/null | tail -1 > gpurun_out/j.json; python -c "import json;d=json.load(open('gpurun_out/j.json'));print(d['value'],d['breakdown_ms'])"
