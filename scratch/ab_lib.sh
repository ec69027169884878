#!/bin/bash
# same-box A/B of two builds of the library (value runs alternate), then a
# launch list of the current build
OUT=gpurun_out; rm -f $OUT/ab.txt
PREV=$PWD/paper_2311_14898_b200/lib/libhongtu_b200_prev.so
for k in 1 2 3; do
  for v in "HT_LIB=$PREV" "HT_X=1"; do
    env $v timeout 300 python bench.py --only-value --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ab.log 2>&1
    echo "[$v] GCN $(grep 'value run' $OUT/ab.log | cut -c1-45)" >> $OUT/ab.txt
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none --csv --log-file $OUT/gcn_launches.csv \
  timeout 600 python bench.py --only-value --steps 1 --warmup 1 --no-cpu-baseline > $OUT/gcn_prof.log 2>&1
