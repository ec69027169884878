# Session-3 A/Bs on one B200: THP-backed pinned host store vs cudaHostAlloc
# (e2e epochs, interleaved), then the GAT row-pass occupancy sweep.
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_epoch.py -q -x -p no:cacheprovider > gpurun_out/d_epoch.log 2>&1; echo "epoch rc=$?"; tail -2 gpurun_out/d_epoch.log
for rep in 1 2; do
  timeout 1200 python bench.py --no-gat --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/d_bench_thp_$rep.json 2> gpurun_out/d_bench_thp_$rep.err; echo "thp rc=$?"
  HT_HOST_ALLOC=cuda timeout 1200 python bench.py --no-gat --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/d_bench_cuda_$rep.json 2> gpurun_out/d_bench_cuda_$rep.err; echo "cuda rc=$?"
done
bash profiles/tools/gat_occupancy_sweep.sh
for rep in 1 2 3; do
  timeout 600 python bench.py --no-gat --only-value --no-cpu-baseline --steps 10 --warmup 3 2>&1 | grep "value run" | sed "s/^/pair $rep /" >> gpurun_out/d_pair_ab.txt
  HT_NO_PAIR=1 timeout 600 python bench.py --no-gat --only-value --no-cpu-baseline --steps 10 --warmup 3 2>&1 | grep "value run" | sed "s/^/nopair $rep /" >> gpurun_out/d_pair_ab.txt
  HT_NO_PAIR=1 HT_NO_MASK_FOLD=1 timeout 600 python bench.py --no-gat --only-value --no-cpu-baseline --steps 10 --warmup 3 2>&1 | grep "value run" | sed "s/^/nopair_nofold $rep /" >> gpurun_out/d_pair_ab.txt
done
cat gpurun_out/d_pair_ab.txt
HT_NO_PAIR=1 timeout 900 python profiles/tools/var_diag.py > gpurun_out/d_phases_nopair.txt 2>&1
timeout 900 python profiles/tools/var_diag.py > gpurun_out/d_phases_pair.txt 2>&1
