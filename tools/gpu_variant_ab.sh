# A/B of a source patch in one box session: A = tree as committed, B = tree + $1 (rebuilt in place)
PATCH=$1
run() { timeout 300 python bench.py --no-cpu --no-e2e --no-loopback --steps 10 2>/dev/null | tail -1 > gpurun_out/ab.json; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$1', d['value'],d['breakdown_ms'])"; }
build() { python -c "import sys; sys.path.insert(0,'.'); from paper_2412_02962_b200 import build as B; B.build()" > /dev/null 2>&1 || echo BUILD FAILED; }
run A
git apply $PATCH 2>/dev/null || patch -p1 < $PATCH > /dev/null; build; run B
patch -R -p1 < $PATCH > /dev/null; build; run A
patch -p1 < $PATCH > /dev/null; build; run B
