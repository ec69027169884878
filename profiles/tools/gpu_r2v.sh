# r2v: narrow-row / piece shape variants, alternating with the default
set -x
for r in 1 2; do
for v in default s_u4 s_u16 s_b8 s_b2 s_m3 up4 up16; do
  if [ $v = default ]; then L=""; else L="paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so"; fi
  HT_LIB=$L timeout 600 python bench.py --only-value --no-gat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2v_${v}_$r.log 2>&1
done
done
for f in gpurun_out/r2v_*.log; do echo "$f $(grep 'value run' $f | cut -c16-45)"; done
