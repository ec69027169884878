# r2t: GCN work-list shape variants (same box A/B, value epochs, two runs each)
set -x
for v in default wl_b8 wl_b32 wl_us2_4 wl_us2_4m3 wl_us1_4 wl_us1_16m3 default; do
  if [ $v = default ]; then L=""; else L="paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so"; fi
  HT_LIB=$L timeout 600 python bench.py --only-value --no-gat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2t_$v.log 2>&1
  echo "$v $(grep 'value run' gpurun_out/r2t_$v.log | cut -c1-60)"
done
