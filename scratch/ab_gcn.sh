#!/bin/bash
OUT=gpurun_out; rm -f $OUT/ab.txt
timeout 900 python -m pytest tests/test_gpu_epoch.py tests/test_gpu_cache.py tests/test_gpu_edges.py -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
PREV=$PWD/paper_2311_14898_b200/lib/libhongtu_b200_prev.so
for k in 1 2; do
  for v in "HT_LIB=$PREV" "HT_X=1"; do
    env $v timeout 300 python bench.py --only-value --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ab.log 2>&1
    echo "[${v:0:6}] GCN $(grep 'value run' $OUT/ab.log | cut -c1-170)" >> $OUT/ab.txt
  done
done
