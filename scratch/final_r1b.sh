#!/bin/bash
# refresh after project-first: bench line, GCN launch list + traffic, cfg3s bench
OUT=gpurun_out
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?" >> $OUT/bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none --csv --log-file $OUT/gcn_launches.csv \
  timeout 600 python bench.py --only-value --steps 1 --warmup 3 --no-cpu-baseline > $OUT/gcn_prof.log 2>&1
timeout 1500 python bench.py --config cfg3s --no-gat > $OUT/bench_cfg3s.json 2> $OUT/bench_cfg3s.err; echo "rc $?" >> $OUT/bench_cfg3s.err
