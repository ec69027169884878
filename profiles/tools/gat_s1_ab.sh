# Same-box A/B of the S1 occupancy (default HT_GAT_S1_MINB=5 vs the
# compiler's choice, variant s1def: python -m paper_2311_14898_b200.build
# --variant s1def HT_GAT_S1_MINB=1) on the cfg-2 GAT sub-line and the cfg5s
# GAT share.
mkdir -p gpurun_out
for rep in 1 2; do
  for v in default s1def; do
    if [ $v = default ]; then lib=paper_2311_14898_b200/lib/libhongtu_b200.so; else lib=paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so; fi
    HT_LIB=$lib timeout 900 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/h_ab_${v}_$rep.json 2> /dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/h_ab_${v}_$rep.json').read().strip().splitlines()[-1]); g=d['gat']; print('cfg2', '$v', $rep, round(d['ms_per_step'],2), round(g['ms_per_step'],2), round(g['edge_kernels']['fwd_ms_per_step'],2), round(g['edge_kernels']['bwd_ms_per_step'],2), round(g['e2e']['ms_per_step'],1))" >> gpurun_out/gat_s1_ab.txt
  done
done
for v in default s1def; do
  if [ $v = default ]; then lib=paper_2311_14898_b200/lib/libhongtu_b200.so; else lib=paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so; fi
  HT_LIB=$lib timeout 1500 python bench.py --config cfg5s --no-gat --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/h_cfg5s_${v}.json 2> /dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/h_cfg5s_${v}.json').read().strip().splitlines()[-1]); print('cfg5s', '$v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],1))" >> gpurun_out/gat_s1_ab.txt
done
cat gpurun_out/gat_s1_ab.txt
