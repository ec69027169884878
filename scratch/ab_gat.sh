#!/bin/bash
OUT=gpurun_out; rm -f $OUT/ab.txt
timeout 900 python -m pytest tests/test_gpu_gat.py tests/test_gpu_cache.py tests/test_gpu_edges.py tests/test_gpu_rank.py -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
PREV=$PWD/paper_2311_14898_b200/lib/libhongtu_b200_prev.so
for k in 1 2; do
  for v in "HT_LIB=$PREV" "HT_X=1"; do
    env $v timeout 300 python bench.py --only-value --kind gat --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ab.log 2>&1
    echo "[${v:0:6}] GAT $(grep -o '"ms_per_step": [0-9.]*' $OUT/ab.log | head -1) $(grep -o '"edge_kernels": {[^}]*}' $OUT/ab.log)" >> $OUT/ab.txt
  done
done
