# Same-box A/B of the GAT row passes' occupancy (minimum resident CTAs per
# SM asked of ptxas): variants built with
#   python -m paper_2311_14898_b200.build --variant s1m5 HT_GAT_S1_MINB=5   (and s1m6, dstm8)
# GAT value epochs on the cfg-2 graph, interleaved twice.
mkdir -p gpurun_out
for rep in 1 2; do
  for v in default s1m5 s1m6 dstm8; do
    if [ $v = default ]; then lib=paper_2311_14898_b200/lib/libhongtu_b200.so; else lib=paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so; fi
    HT_LIB=$lib timeout 600 python bench.py --only-value --kind gat --no-cpu-baseline --steps 5 --warmup 3 2>&1 | grep "GAT:" | sed "s/^/$v $rep /" >> gpurun_out/gat_occ_sweep.txt
  done
done
cat gpurun_out/gat_occ_sweep.txt
