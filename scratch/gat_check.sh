#!/bin/bash
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_gat.py -x -q > $OUT/pytest_gat.log 2>&1; echo "rc $?" >> $OUT/pytest_gat.log
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_gat.py -x -q -k "oracle and 2-3" > $OUT/memcheck_gat.log 2>&1; echo "rc $?" >> $OUT/memcheck_gat.log
