# Session-3 GEMM changes on one B200: the GEMM unit tests first (short
# timeout: a CTA-pair barrier bug would hang), the mask-fold epoch test,
# then the cfg-2 line, the value-epoch launch list and the GPU suite.
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider > gpurun_out/b_gemm.log 2>&1; echo "gemm rc=$?"; tail -3 gpurun_out/b_gemm.log
timeout 300 python -m pytest tests/test_gpu_cache.py -q -x -k mask_fold -p no:cacheprovider > gpurun_out/b_fold.log 2>&1; echo "fold rc=$?"; tail -3 gpurun_out/b_fold.log
grep -q "passed" gpurun_out/b_gemm.log || exit 1
timeout 1200 python bench.py --no-gat > gpurun_out/b_bench_cfg2.json 2> gpurun_out/b_bench_cfg2.err; echo "cfg2 rc=$?"
HT_NO_PAIR=1 timeout 1200 python bench.py --no-gat --only-value --no-cpu-baseline > gpurun_out/b_bench_cfg2_nopair.json 2> gpurun_out/b_bench_cfg2_nopair.err; echo "cfg2 nopair rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none --csv --log-file gpurun_out/b_value_launches.csv python bench.py --profile-epoch value --steps 1 --warmup 2 > gpurun_out/b_ncu_list.log 2>&1; echo "ncu rc=$?"
python profiles/summarize_launches.py gpurun_out/b_value_launches.csv > gpurun_out/b_value_launches.txt
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_tc_gemm -c 3 \
    -o gpurun_out/b_tc_gemm python bench.py --profile-epoch value --steps 1 --warmup 2 > gpurun_out/b_ncu_gemm.log 2>&1; echo "ncu2 rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/b_gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/b_gputest.log
