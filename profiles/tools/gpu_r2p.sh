# r2p: K-tail k-step skip - GEMM unit/epoch parity, rates, value epoch
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_epoch.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r2p_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2p_tests.log
timeout 600 python profiles/tools/tf32_peak.py > gpurun_out/r2p_rates.json 2>&1; echo "rates rc=$?"; grep -A2 "z_relu_3xtf32_k100" gpurun_out/r2p_rates.json
timeout 600 python bench.py --only-value --no-gat --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep "value run"
