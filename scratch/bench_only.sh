#!/bin/bash
OUT=gpurun_out
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?" >> $OUT/bench.err
