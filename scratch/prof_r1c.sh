#!/bin/bash
# r1 refresh: launch lists (GCN, GAT), full captures of the top kernels, cfg3s bench line
OUT=gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none --csv --log-file $OUT/gcn_launches.csv \
  timeout 600 python bench.py --only-value --steps 1 --warmup 3 --no-cpu-baseline > $OUT/gcn_prof.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file $OUT/gat_launches.csv \
  timeout 600 python bench.py --only-value --kind gat --steps 1 --warmup 1 --no-cpu-baseline > $OUT/gat_prof.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_tc_wgrad" -s 2 -c 1 -o $OUT/full_wgrad -f \
  timeout 600 python bench.py --only-value --steps 1 --warmup 1 --no-cpu-baseline > $OUT/full_wgrad.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_seg_gather_v4" -s 2 -c 1 -o $OUT/full_seg -f \
  timeout 600 python bench.py --only-value --steps 1 --warmup 1 --no-cpu-baseline > $OUT/full_seg.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_tc_gemm" -s 40 -c 1 -o $OUT/full_gemm -f \
  timeout 600 python bench.py --only-value --steps 1 --warmup 1 --no-cpu-baseline > $OUT/full_gemm.log 2>&1
timeout 1500 python bench.py --config cfg3s --no-gat > $OUT/bench_cfg3s.json 2> $OUT/bench_cfg3s.err; echo "rc $?" >> $OUT/bench_cfg3s.err
