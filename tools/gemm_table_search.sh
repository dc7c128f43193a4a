#!/bin/bash
# In-step search over the GEMM configuration table: for each hot shape key and candidate
# (bn splits pair), run the 1024^2 bench with that one table entry replaced; baselines interleaved.
cd $GRAFT_REPO_ROOT
B="--steps 10 --warmup 3 --no-cpu --no-large --no-xf --no-loopback --no-e2e --no-profile"
python paper_2412_02962_b200/build.py > /dev/null 2>&1 || echo BUILD FAILED
T=profiles/gemm_tune_b200.txt
val() { PCPP_TUNE_FILE=$1 timeout 300 python bench.py $B 2>/dev/null | tail -1 | python -c "import json,sys;print(json.load(sys.stdin)['value'])"; }
echo "base $(val $T)"
while IFS='|' read -r key cands; do
  for c in $cands; do
    cfg=${c//,/ }
    awk -v k="$key" -v c="$cfg" '{ if (index($0, k " ") == 1 && NF == 15) print k " " c; else print }' $T > gpurun_out/tt.txt
    echo "[$key] -> $cfg : $(val gpurun_out/tt.txt)"
  done
  echo "base $(val $T)"
done <<'LIST'
32 32 2 3840 1280 1280 1 1 1280 0 1 0|256,1,0 160,1,1 128,1,1
32 32 2 1280 1280 1280 1 1 0 1 1 0|256,1,0 256,1,1 128,1,1 160,1,1
32 32 2 1280 1280 1280 9 1 0 0 1 1|256,1,1 160,1,1
64 64 2 640 640 640 1 1 0 1 1 0|128,1,0 128,1,1
64 64 2 1920 640 640 1 1 640 0 1 0|128,1,1 160,1,1
LIST
