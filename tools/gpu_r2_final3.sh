#!/bin/bash
# round-2 final evidence (session 3): the driver's GPU suite, smoke, default bench (N = 1), reference
# arm, the N = 2 code path on one GPU, one-step launch lists (n = 1, n = 8), ncu --set full of the
# top kernels, compute-sanitizer incl. the new kernels
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1
timeout 2400 python -m pytest tests/ -x -q -m gpu > gpurun_out/g_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/g_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g_smoke.log
timeout 900 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo "bench rc=$?" >> gpurun_out/g_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/g_bench_ref.json 2> gpurun_out/g_bench_ref.err; echo "ref rc=$?" >> gpurun_out/g_bench_ref.err
PCPP_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/g_bench2.json 2> gpurun_out/g_bench2.err; echo "bench2 rc=$?" >> gpurun_out/g_bench2.err
PROF_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_n1.csv python tools/prof_step.py 1 128 sdxl 1 > gpurun_out/g_prof_n1.out 2>&1
PROF_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_n8.csv python tools/prof_step.py 8 128 sdxl 1 > gpurun_out/g_prof_n8.out 2>&1
for spec in "gemm_tc_kernel:20" "gemm_tc2_kernel:5" "attn_tc_kernel:30" "attn_tc_kernel:65" "gn_apply_bulk:10" "gn_stats_kernel:8" "conv_out_mma:0" "conv_in_kernel:0"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/g_full_${k}_$s python tools/prof_step.py 1 128 sdxl 1 > /dev/null 2>&1
done
timeout 1500 bash tools/gpu_sanitize.sh > gpurun_out/g_sanitizer.txt 2>&1
echo "== memcheck attention tail split (level-1 / level-2 geometry, op entry)" >> gpurun_out/g_sanitizer.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_fullsize.py -q -k attention 2>&1 | grep -E "ERROR SUMMARY|passed|failed" >> gpurun_out/g_sanitizer.txt
tail -n 3 gpurun_out/g_gpu.log gpurun_out/g_smoke.log gpurun_out/g_bench.err gpurun_out/g_bench_ref.err gpurun_out/g_bench2.err; grep -E "ERROR SUMMARY|==" gpurun_out/g_sanitizer.txt | head -30
