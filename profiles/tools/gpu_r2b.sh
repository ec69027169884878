# r2b: work-list aggregation + single-launch GEMM - parity, A/B, launch list, counters
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_worklist.py tests/test_gpu_epoch.py -x -q -p no:cacheprovider > gpurun_out/r2b_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2b_tests.log
for v in 0 1; do
  HT_SEG_SPLIT_LAUNCH=$v timeout 600 python bench.py --only-value --no-gat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_ab_$v.log 2>&1
  grep "value run" gpurun_out/r2b_ab_$v.log
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r2b_value_launches.csv python bench.py --profile-epoch value --steps 1 --warmup 2 > gpurun_out/r2b_ncu_value.log 2>&1; echo "ncu rc=$?"
python profiles/summarize_launches.py gpurun_out/r2b_value_launches.csv > gpurun_out/r2b_value_launches.txt 2>&1; head -30 gpurun_out/r2b_value_launches.txt
timeout 900 ncu --replay-mode app-range --profile-from-start off --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_pcie_e2e.csv python bench.py --profile-epoch e2e --steps 1 --warmup 2 > gpurun_out/r2b_pcie_e2e.log 2>&1; echo "pcie e2e rc=$?"; tail -5 gpurun_out/r2b_pcie_e2e.csv; tail -2 gpurun_out/r2b_pcie_e2e.log
timeout 900 ncu --replay-mode app-range --profile-from-start off --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_pcie_virt.csv python bench.py --profile-epoch virt --steps 1 --warmup 1 > gpurun_out/r2b_pcie_virt.log 2>&1; echo "pcie virt rc=$?"; tail -5 gpurun_out/r2b_pcie_virt.csv; tail -2 gpurun_out/r2b_pcie_virt.log
timeout 600 python profiles/tools/tf32_peak.py > gpurun_out/r2b_tf32_peak.json 2> gpurun_out/r2b_tf32_peak.err; echo "tf32 rc=$?"; cat gpurun_out/r2b_tf32_peak.json | head -40
timeout 900 python -m pytest tests/test_gpu_cache.py -x -q -p no:cacheprovider > gpurun_out/r2b_cache.log 2>&1; echo "cache tests rc=$?"; tail -15 gpurun_out/r2b_cache.log
