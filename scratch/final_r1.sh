#!/bin/bash
# round-end refresh: full GPU suite, smoke, bench line, launch lists (GCN, GAT)
OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?" >> $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?" >> $OUT/bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none --csv --log-file $OUT/gcn_launches.csv \
  timeout 600 python bench.py --only-value --steps 1 --warmup 3 --no-cpu-baseline > $OUT/gcn_prof.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file $OUT/gat_launches.csv \
  timeout 600 python bench.py --only-value --kind gat --steps 1 --warmup 1 --no-cpu-baseline > $OUT/gat_prof.log 2>&1
