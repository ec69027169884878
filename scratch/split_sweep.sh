#!/bin/bash
OUT=gpurun_out
rm -f $OUT/split.txt
for v in 4096 2048 1024 512; do
  HT_SPLIT=$v timeout 300 python bench.py --only-value --steps 5 --warmup 3 --no-cpu-baseline > $OUT/split_gcn_$v.log 2>&1
  echo "split=$v GCN $(grep 'value run' $OUT/split_gcn_$v.log | cut -c1-60)" >> $OUT/split.txt
  HT_SPLIT=$v timeout 300 python bench.py --only-value --kind gat --steps 5 --warmup 3 --no-cpu-baseline > $OUT/split_gat_$v.log 2>&1
  echo "split=$v GAT $(grep -o '"ms_per_step": [0-9.]*' $OUT/split_gat_$v.log | head -1)" >> $OUT/split.txt
done
