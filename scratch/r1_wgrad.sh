#!/bin/bash
OUT=gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > $OUT/pytest_gemm.log 2>&1; rc=$?; echo "gemm rc $rc" >> $OUT/pytest_gemm.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --no-gat > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?" >> $OUT/bench.err
