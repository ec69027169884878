# r2i: GAT split backward parity + A/B, memcheck (leaks), cfg4s with allocation trace
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gat.py tests/test_gpu_fullsize.py::test_fullsize_gat_layerwise_vs_fp64_oracle tests/test_gpu_cache.py tests/test_gpu_rank.py -x -q -p no:cacheprovider > gpurun_out/r2i_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2i_tests.log
for v in 0 1; do
  HT_NO_GAT_SPLIT=$v timeout 900 python bench.py --only-value --kind gat --steps 5 --warmup 3 > gpurun_out/r2i_gat_$v.log 2>&1
  grep "GAT:" gpurun_out/r2i_gat_$v.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l.split('GAT: ',1)[1]); print('split_off=$v', round(d['ms_per_step'],2), round(d['edge_kernels']['fwd_ms_per_step'],2), round(d['edge_kernels']['bwd_ms_per_step'],2), round(d['e2e']['ms_per_step'],1))"
done
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python profiles/tools/sanitize_epoch.py > gpurun_out/r2i_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r2i_memcheck.log
HT_TRACE_CACHE=1 timeout 2400 python bench.py --config cfg4s --no-gat --steps 3 --warmup 3 > gpurun_out/r2i_bench_cfg4s.json 2> gpurun_out/r2i_bench_cfg4s.err; echo "cfg4s rc=$?"; grep "^\[bench\]\|^\[ht\]" gpurun_out/r2i_bench_cfg4s.err; tail -1 gpurun_out/r2i_bench_cfg4s.err
