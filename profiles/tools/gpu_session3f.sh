set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider > gpurun_out/f_gemm.log 2>&1; echo "gemm rc=$?"; tail -1 gpurun_out/f_gemm.log
bash profiles/tools/gat_occupancy_ab.sh
bash profiles/tools/gpu_session3e.sh
