# Top-layer mask folded into the loss kernel: the epoch tests, the GPU
# suite, a same-box A/B against HT_NO_MASK_FOLD=1, and the cfg-2 line.
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_cache.py tests/test_gpu_epoch.py -q -x -p no:cacheprovider > gpurun_out/i_quick.log 2>&1; echo "quick rc=$?"; tail -1 gpurun_out/i_quick.log
grep -q " passed" gpurun_out/i_quick.log && ! grep -q "failed" gpurun_out/i_quick.log || exit 1
for rep in 1 2 3; do
  timeout 600 python bench.py --no-gat --only-value --no-cpu-baseline --steps 10 --warmup 3 2>&1 | grep "value run" | sed "s/^/fold $rep /" >> gpurun_out/i_fold_ab.txt
  HT_NO_MASK_FOLD=1 timeout 600 python bench.py --no-gat --only-value --no-cpu-baseline --steps 10 --warmup 3 2>&1 | grep "value run" | sed "s/^/nofold $rep /" >> gpurun_out/i_fold_ab.txt
done
cat gpurun_out/i_fold_ab.txt | cut -c1-50
timeout 1200 python bench.py > gpurun_out/i_bench_cfg2.json 2> gpurun_out/i_bench_cfg2.err; echo "cfg2 rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/i_gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/i_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/i_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/i_smoke.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none --csv --log-file gpurun_out/i_value_launches.csv python bench.py --profile-epoch value --steps 1 --warmup 2 > gpurun_out/i_ncu_list.log 2>&1; echo "ncu rc=$?"
python profiles/summarize_launches.py gpurun_out/i_value_launches.csv > gpurun_out/i_value_launches.txt
