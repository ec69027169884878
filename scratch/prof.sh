#!/bin/bash
# profiling helper run on the GPU box: launch list of one HBM-resident epoch
# run + full captures of the named kernels
set -x
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file $OUT/launches.csv \
  timeout 600 python bench.py --only-value --steps 1 --warmup 3 --no-cpu-baseline > $OUT/prof_bench.log 2>&1
for K in "$@"; do
  tag=$(echo "$K" | tr -c 'a-zA-Z0-9' '_')
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$K" -s 2 -c 1 -o $OUT/full_$tag -f \
    timeout 600 python bench.py --only-value --steps 1 --warmup 1 --no-cpu-baseline > $OUT/full_$tag.log 2>&1
done
