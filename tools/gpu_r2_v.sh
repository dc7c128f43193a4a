#!/bin/bash
# round-2 V(2): out-projection started early behind its attention (row flags) -- correctness (ops, path,
# golden, peer, xf), same-box A/B against PCPP_EARLY_START=0
cd $GRAFT_REPO_ROOT
python paper_2412_02962_b200/build.py > gpurun_out/w_build.log 2>&1
B="--steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e"
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x > gpurun_out/w_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/w_ops.log
for i in 1 2; do
  PCPP_EARLY_START=0 timeout 600 python bench.py $B > gpurun_out/w_off$i.json 2> gpurun_out/w_off$i.err
  timeout 600 python bench.py $B > gpurun_out/w_on$i.json 2> gpurun_out/w_on$i.err
done
for f in w_off1 w_on1 w_off2 w_on2; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['value'],d['breakdown_ms'])"; done
timeout 2400 python -m pytest tests/test_gpu_path.py tests/test_gpu_golden.py tests/test_gpu_peer.py tests/test_gpu_xf.py tests/test_gpu_fullsize.py -q -x > gpurun_out/w_path.log 2>&1; echo "path rc=$?" >> gpurun_out/w_path.log
tail -n 3 gpurun_out/w_ops.log gpurun_out/w_path.log
