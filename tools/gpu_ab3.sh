bash tools/gpu_variant_ab.sh tools/variant_exp25.patch
bash tools/gpu_variant_ab.sh tools/variant_exp12.patch 2>&1 | grep B
git apply tools/variant_exp25.patch; python -c "import sys; sys.path.insert(0,'.'); from paper_2412_02962_b200 import build as B; B.build()" >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py tests/test_gpu_path.py -m gpu -q -x -k "attention or path_matches" 2>&1 | tail -2
