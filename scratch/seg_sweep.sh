#!/bin/bash
OUT=gpurun_out
for v in 0 1 2 3 4 5 6 7; do
  HT_SEG_VARIANT1=$v timeout 300 python bench.py --only-value --steps 5 --warmup 3 --no-cpu-baseline > $OUT/sweep1_$v.log 2>&1
  echo "v1=$v $(grep 'value run' $OUT/sweep1_$v.log)" >> $OUT/sweep.txt
done
