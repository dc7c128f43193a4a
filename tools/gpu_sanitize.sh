for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  PCPP_AUTOTUNE=0 timeout 900 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_tiny.py 2>&1 | grep -v "^========= Saved host\|Host Frame" | tail -12
done
for f in "160,1,1" "256,1,1" "64,2,0" "160,1,2" "128,1,4"; do
  echo "== memcheck sdxl 32x32 n=2, GEMM forced $f"
  PCPP_AUTOTUNE=0 PCPP_GEMM_FORCE=$f timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python tools/sanitize_tiny.py sdxl 2>&1 | grep -v "^========= Saved host\|Host Frame" | tail -4
done
