# r2u: combined work-list shape variants, alternating with the default (noise ~0.3 ms)
set -x
for r in 1 2; do
for v in default c1 c2 c3; do
  if [ $v = default ]; then L=""; else L="paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so"; fi
  HT_LIB=$L timeout 600 python bench.py --only-value --no-gat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2u_${v}_$r.log 2>&1
  echo "$v $r $(grep 'value run' gpurun_out/r2u_${v}_$r.log | cut -c1-50)"
done
done
