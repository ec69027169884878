#!/bin/bash
OUT=gpurun_out; rm -f $OUT/sweep.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
HT_SEG_VARIANT=9 HT_SEG_VARIANT1=9 timeout 600 python -m pytest tests/test_gpu_epoch.py tests/test_gpu_cache.py tests/test_gpu_edges.py tests/test_gpu_comm.py -x -q > $OUT/pytest_stream.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_stream.log
for v in "0 0" "8 8" "9 9" "10 10" "0 0" "9 9" "8 9" "9 10"; do
  set -- $v
  HT_SEG_VARIANT=$1 HT_SEG_VARIANT1=$2 timeout 300 python bench.py --only-value --steps 5 --warmup 3 --no-cpu-baseline > $OUT/sw.log 2>&1
  echo "[$1 $2] $(grep 'value run' $OUT/sw.log | cut -c1-300)" >> $OUT/sweep.txt
done
