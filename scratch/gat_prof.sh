#!/bin/bash
OUT=gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none --csv --log-file $OUT/gat_launches.csv \
  timeout 600 python bench.py --only-value --kind gat --steps 1 --warmup 1 --no-cpu-baseline > $OUT/gat_prof.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_gat_src" -s 4 -c 1 -o $OUT/full_gat_src -f \
  timeout 600 python bench.py --only-value --kind gat --steps 1 --warmup 1 --no-cpu-baseline > $OUT/full_gat.log 2>&1
