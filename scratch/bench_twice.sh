#!/bin/bash
OUT=gpurun_out
for k in 1 2; do
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_$k.json 2> $OUT/bench_$k.err
done
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc $?" >> $OUT/pytest_gpu.log
