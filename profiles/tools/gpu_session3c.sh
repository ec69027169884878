# Session-3 GEMM changes on one B200: the GEMM unit tests first (short
# timeout: a CTA-pair barrier bug would hang), the mask-fold epoch test,
# then the cfg-2 line, the value-epoch launch list and the GPU suite.
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider > gpurun_out/c_gemm.log 2>&1; echo "gemm rc=$?"; tail -3 gpurun_out/c_gemm.log
timeout 300 python -m pytest tests/test_gpu_cache.py -q -x -k mask_fold -p no:cacheprovider > gpurun_out/c_fold.log 2>&1; echo "fold rc=$?"; tail -3 gpurun_out/c_fold.log
grep -q "passed" gpurun_out/c_gemm.log || exit 1
timeout 1200 python bench.py > gpurun_out/c_bench_cfg2.json 2> gpurun_out/c_bench_cfg2.err; echo "cfg2 rc=$?"
HT_NO_PAIR=1 timeout 1200 python bench.py --no-gat --only-value --no-cpu-baseline > gpurun_out/c_bench_cfg2_nopair.json 2> gpurun_out/c_bench_cfg2_nopair.err; echo "cfg2 nopair rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none --csv --log-file gpurun_out/c_value_launches.csv python bench.py --profile-epoch value --steps 1 --warmup 2 > gpurun_out/c_ncu_list.log 2>&1; echo "ncu rc=$?"
python profiles/summarize_launches.py gpurun_out/c_value_launches.csv > gpurun_out/c_value_launches.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/c_gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/c_gputest.log
timeout 1500 python bench.py --config cfg4s --no-gat --steps 3 --warmup 3 > gpurun_out/c_bench_cfg4s.json 2> gpurun_out/c_bench_cfg4s.err; echo "cfg4s rc=$?"
