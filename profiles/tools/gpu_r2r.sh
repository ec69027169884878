# r2r: GAT destination work list - parity, launch list, value
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gat.py tests/test_gpu_cache.py tests/test_gpu_rank.py -x -q -p no:cacheprovider > gpurun_out/r2r_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2r_tests.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2r_gat_launches.csv python bench.py --profile-epoch value --kind gat --steps 1 --warmup 2 > gpurun_out/r2r_gat_ncu.log 2>&1; echo "ncu rc=$?"
python profiles/summarize_launches.py gpurun_out/r2r_gat_launches.csv > gpurun_out/r2r_gat_launches.txt 2>&1; head -10 gpurun_out/r2r_gat_launches.txt
timeout 900 python bench.py --only-value --kind gat --steps 5 --warmup 3 > gpurun_out/r2r_gat.log 2>&1; grep "GAT:" gpurun_out/r2r_gat.log | cut -c150-330
