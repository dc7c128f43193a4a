# L2 1x1 GEMM shapes (M = 2048 tokens): graph-timed config sweep + one ncu full capture
for shape in "32 32 1280 1280 1 1" "32 32 1280 1280 1 1 1" "32 32 1280 3840 1 1" "64 64 640 640 1 1" "64 64 640 1920 1 1"; do
  echo "== $shape"
  python tools/bench_gemm.py $shape
  for f in "128,1,0" "160,1,0" "256,1,0" "128,2,0" "160,2,0" "256,2,0" "256,1,1" "128,1,1" "160,1,1" "256,2,1" "128,4,0"; do
    PCPP_GEMM_FORCE=$f timeout 60 python tools/bench_gemm.py $shape 2>&1 | tail -1
  done
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 27 -c 1 -o gpurun_out/r1f_gemm_l2_27 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile --no-loopback > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r1f_gemm_l2_27.ncu-rep
