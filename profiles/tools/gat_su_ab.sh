# Same-box A/B of S1 with 4 CSR rows in flight at 6 / 8 CTAs per SM
# (variants: --variant su4m6 HT_GAT_SU=4 HT_GAT_S1_MINB=6, su4m8 ... =8)
# against the default (8 rows in flight, 5 CTAs per SM), cfg-2 GAT sub-line.
mkdir -p gpurun_out
for rep in 1 2; do
  for v in default su4m6 su4m8; do
    if [ $v = default ]; then lib=paper_2311_14898_b200/lib/libhongtu_b200.so; else lib=paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so; fi
    HT_LIB=$lib timeout 900 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/k_ab_${v}_$rep.json 2> /dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/k_ab_${v}_$rep.json').read().strip().splitlines()[-1]); g=d['gat']; print('cfg2', '$v', $rep, round(d['ms_per_step'],2), round(g['ms_per_step'],2), round(g['edge_kernels']['fwd_ms_per_step'],2), round(g['edge_kernels']['bwd_ms_per_step'],2), round(g['e2e']['ms_per_step'],1))" >> gpurun_out/gat_su_ab.txt
  done
done
for v in default su4m6 su4m8; do
  if [ $v = default ]; then lib=paper_2311_14898_b200/lib/libhongtu_b200.so; else lib=paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so; fi
  HT_LIB=$lib timeout 1500 python bench.py --config cfg5s --no-gat --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/k_cfg5s_${v}.json 2> /dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/k_cfg5s_${v}.json').read().strip().splitlines()[-1]); print('cfg5s', '$v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],1))" >> gpurun_out/gat_su_ab.txt
done
cat gpurun_out/gat_su_ab.txt
