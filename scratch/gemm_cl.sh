#!/bin/bash
OUT=gpurun_out; rm -f $OUT/ab.txt
timeout 180 python -m pytest tests/test_gpu_gemm.py -x -q > $OUT/pytest_gemm.log 2>&1; rc=$?; echo "gemm rc $rc" >> $OUT/pytest_gemm.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
for k in 1 2; do
  for v in "HT_GEMM_NO_CLUSTER=1" "HT_X=1"; do
    env $v timeout 300 python bench.py --only-value --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ab.log 2>&1
    echo "[$v] GCN $(grep 'value run' $OUT/ab.log | cut -c1-200)" >> $OUT/ab.txt
    env $v timeout 300 python bench.py --only-value --kind gat --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ab.log 2>&1
    echo "[$v] GAT $(grep -o '"ms_per_step": [0-9.]*' $OUT/ab.log | head -1)" >> $OUT/ab.txt
  done
done
