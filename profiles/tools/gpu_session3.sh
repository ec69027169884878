# Session-3 check on one B200: the GPU suite, the cfg-2 contract line, and
# full ncu captures of the two largest GAT kernels (outputs in gpurun_out/).
set -x
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/a_bench_cfg2.json 2> gpurun_out/a_bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_gat_bwd_s1_work -c 1 \
    -o gpurun_out/gat_s1 python bench.py --profile-epoch value --kind gat --steps 1 --warmup 2 > gpurun_out/gat_s1.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_gat_dst -c 1 \
    -o gpurun_out/gat_dst python bench.py --profile-epoch value --kind gat --steps 1 --warmup 2 > gpurun_out/gat_dst.log 2>&1; echo "ncu rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/a_gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/a_gputest.log
