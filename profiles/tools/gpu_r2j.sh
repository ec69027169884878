# r2j: GAT launch lists (split vs fused backward), GAT tests, cfg4s with the cross-epoch plan fix
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gat.py tests/test_gpu_cache.py -x -q -p no:cacheprovider > gpurun_out/r2j_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2j_tests.log
for v in 0 1; do
  HT_NO_GAT_SPLIT=$v timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/r2j_gat_launches_$v.csv python bench.py --profile-epoch value --kind gat --steps 1 --warmup 2 > gpurun_out/r2j_gat_ncu_$v.log 2>&1; echo "ncu $v rc=$?"
  python profiles/summarize_launches.py gpurun_out/r2j_gat_launches_$v.csv > gpurun_out/r2j_gat_launches_$v.txt 2>&1; head -22 gpurun_out/r2j_gat_launches_$v.txt
done
HT_TRACE_CACHE=1 timeout 2400 python bench.py --config cfg4s --no-gat --steps 3 --warmup 3 > gpurun_out/r2j_bench_cfg4s.json 2> gpurun_out/r2j_bench_cfg4s.err; echo "cfg4s rc=$?"; grep "^\[bench\]\|^\[ht\]" gpurun_out/r2j_bench_cfg4s.err | sort | uniq -c | head; tail -1 gpurun_out/r2j_bench_cfg4s.err
