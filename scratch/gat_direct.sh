#!/bin/bash
OUT=gpurun_out; rm -f $OUT/ab.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?" >> $OUT/smoke.log
for k in 1 2; do
  for v in "HT_NO_GAT_DIRECT=1" "HT_X=1"; do
    env $v timeout 300 python bench.py --only-value --kind gat --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ab.log 2>&1
    echo "[$v] GAT $(grep -o '"ms_per_step": [0-9.]*' $OUT/ab.log | head -1) $(grep -o '"value": [0-9.]*' $OUT/ab.log | head -1)" >> $OUT/ab.txt
  done
done
