# r2d: column-sliced work-list aggregation - parity vs split launch, value A/B, launch list
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_worklist.py -x -q -p no:cacheprovider > gpurun_out/r2d_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2d_tests.log
for v in 0 32 64; do
  HT_COL_SLICE=$v timeout 600 python bench.py --only-value --no-gat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_ab_$v.log 2>&1
  grep "value run" gpurun_out/r2d_ab_$v.log
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r2d_value_launches.csv python bench.py --profile-epoch value --steps 1 --warmup 2 > gpurun_out/r2d_ncu_value.log 2>&1; echo "ncu rc=$?"
python profiles/summarize_launches.py gpurun_out/r2d_value_launches.csv > gpurun_out/r2d_value_launches.txt 2>&1; head -30 gpurun_out/r2d_value_launches.txt
