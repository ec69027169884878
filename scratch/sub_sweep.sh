#!/bin/bash
OUT=gpurun_out; rm -f $OUT/sweep.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
for v in "HT_NO_SUBWARP=1" "HT_SUB_VARIANT=0" "HT_SUB_VARIANT=1" "HT_SUB_VARIANT=2" "HT_SUB_VARIANT=3" "HT_NO_SUBWARP=1" "HT_SUB_VARIANT=0"; do
  env $v timeout 300 python bench.py --only-value --steps 5 --warmup 3 --no-cpu-baseline > $OUT/sw.log 2>&1
  echo "[$v] $(grep 'value run' $OUT/sw.log | cut -c1-300)" >> $OUT/sweep.txt
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none --csv --log-file $OUT/gcn_launches.csv \
  timeout 600 python bench.py --only-value --steps 1 --warmup 1 --no-cpu-baseline > $OUT/gcn_prof.log 2>&1
