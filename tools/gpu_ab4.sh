bash tools/gpu_variant_ab.sh $1
git apply $1 2>/dev/null; python -c "import sys; sys.path.insert(0,'.'); from paper_2412_02962_b200 import build as B; B.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
