#!/bin/bash
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_gat.py -x -q > $OUT/pytest_gat.log 2>&1; echo "rc $?" >> $OUT/pytest_gat.log
timeout 600 python scratch/gat_diag.py > $OUT/gat_diag.log 2>&1; echo "rc $?" >> $OUT/gat_diag.log
DIAG_KIND=gcn timeout 600 python scratch/gat_diag.py > $OUT/gcn_diag.log 2>&1; echo "rc $?" >> $OUT/gcn_diag.log
