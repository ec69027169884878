# r2s: GAT rows-in-flight variants on the work-list kernels (same box A/B)
set -x
for v in default gat_du8 gat_du2 gat_su16 gat_su4; do
  if [ $v = default ]; then L=""; else L="paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so"; fi
  HT_LIB=$L timeout 900 python bench.py --only-value --kind gat --steps 5 --warmup 3 > gpurun_out/r2s_gat_$v.log 2>&1
  grep "GAT:" gpurun_out/r2s_gat_$v.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l.split('GAT: ',1)[1]); print('$v', round(d['ms_per_step'],2), round(d['edge_kernels']['fwd_ms_per_step'],2), round(d['edge_kernels']['bwd_ms_per_step'],2))"
done
