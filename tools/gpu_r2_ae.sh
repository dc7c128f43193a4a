#!/bin/bash
# round-2 AE: GroupNorm apply grid -- stages per CTA 1 / 2 / 3 / 4 (fewer CTAs for small tensors)
cd $GRAFT_REPO_ROOT
B="--steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e"
python paper_2412_02962_b200/build.py > /dev/null 2>&1 || echo BUILD FAILED
for rep in 1 2; do for v in 148 222 296; do
  PCPP_GN_CAP=$v timeout 600 python bench.py $B 2>/dev/null | tail -1 > gpurun_out/ae_$v.json; python -c "import json;d=json.load(open('gpurun_out/ae_$v.json'));print('cap$v', d['value'],d['breakdown_ms'])"
done; done
