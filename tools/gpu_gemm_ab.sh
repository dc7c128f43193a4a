for shape in "128 128 320 320 9 1" "64 64 640 640 9 1" "32 32 1280 1280 9 1" "64 64 640 640 1 1"; do
for f in "" "160,1,0" "160,1,1" "128,1,1" "64,1,0" "256,1,1" "128,1,0"; do
  PCPP_GEMM_FORCE=$f timeout 60 python tools/bench_gemm.py $shape 2>&1 | tail -1
done; done
