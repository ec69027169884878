# r2g: GAT record packing + one-device buffers: parity, GAT A/B, cfg4s line, sanitizers
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gat.py tests/test_gpu_cache.py tests/test_gpu_epoch.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r2g_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2g_tests.log
timeout 900 python bench.py --only-value --kind gat --steps 5 --warmup 3 > gpurun_out/r2g_gat.log 2>&1; grep "GAT" gpurun_out/r2g_gat.log | cut -c1-600
timeout 2400 python bench.py --config cfg4s --no-gat --steps 3 --warmup 3 > gpurun_out/r2g_bench_cfg4s.json 2> gpurun_out/r2g_bench_cfg4s.err; echo "cfg4s rc=$?"; tail -3 gpurun_out/r2g_bench_cfg4s.err
bash profiles/tools/gpu_r2f.sh
