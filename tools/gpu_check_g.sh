for i in 1 2 3; do timeout 200 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench_g.log 2>&1; echo "rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bench_g.log').read().strip().splitlines()[-1]);print(d['value'],d['breakdown_ms'])"; done
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py tests/test_gpu_path.py -m gpu -q -x 2>&1 | tail -2
for shape in "128 128 320 320 9 1" "32 32 1280 1280 1 1"; do for f in "160,1,0" "128,1,0"; do PCPP_GEMM_FORCE=$f timeout 60 python tools/bench_gemm.py $shape 2>&1 | tail -1; done; done
