set -x
mkdir -p gpurun_out
for r in 1 2; do
for v in default g_s1b4 g_s1b16 g_db4 g_db16; do
  if [ $v = default ]; then L=""; else L="paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so"; fi
  HT_LIB=$L timeout 900 python bench.py --only-value --kind gat --steps 5 --warmup 3 > gpurun_out/gs_${v}_$r.log 2>&1
done
done
