#!/bin/bash
# clean re-sweep of the aggregation variants (after the SGD stall fix)
OUT=gpurun_out; rm -f $OUT/sweep.txt
for v in 0 1 2 3 4 5 6 7 0; do
  HT_SEG_VARIANT=$v timeout 300 python bench.py --only-value --steps 5 --warmup 3 --no-cpu-baseline > $OUT/sw.log 2>&1
  echo "[wide $v] $(grep 'value run' $OUT/sw.log | cut -c1-170)" >> $OUT/sweep.txt
done
for v in 0 1 2 3 4 5 6 7 0; do
  HT_SEG_VARIANT1=$v timeout 300 python bench.py --only-value --steps 5 --warmup 3 --no-cpu-baseline > $OUT/sw.log 2>&1
  echo "[narrow $v] $(grep 'value run' $OUT/sw.log | cut -c1-170)" >> $OUT/sweep.txt
done
