# Session-3 contract lines of the per-GPU shares with the final code.
set -x
mkdir -p gpurun_out
for c in cfg3s cfg4s cfg5s; do timeout 2400 python bench.py --config $c --no-gat --steps 3 --warmup 3 > gpurun_out/j_bench_$c.json 2> gpurun_out/j_bench_$c.err; echo "$c rc=$?"; done
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_tc_gemm -c 1 \
    -o gpurun_out/j_tc_gemm python bench.py --profile-epoch value --steps 1 --warmup 2 > gpurun_out/j_ncu_gemm.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_gat_dst -c 1 \
    -o gpurun_out/j_gat_dst python bench.py --profile-epoch value --kind gat --steps 1 --warmup 2 > gpurun_out/j_ncu_gat.log 2>&1; echo "ncu gat rc=$?"
