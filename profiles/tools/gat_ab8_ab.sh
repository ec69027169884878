# Same-box A/B of the GAT split-backward destination passes A / B at 8 CTAs
# per SM (variant: --variant ab8 HT_GAT_AB_MINB=8) against the default,
# cfg-2 GAT sub-line.
mkdir -p gpurun_out
for rep in 1 2; do
  for v in default ab8; do
    if [ $v = default ]; then lib=paper_2311_14898_b200/lib/libhongtu_b200.so; else lib=paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so; fi
    HT_LIB=$lib timeout 900 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/l_ab_${v}_$rep.json 2> /dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/l_ab_${v}_$rep.json').read().strip().splitlines()[-1]); g=d['gat']; print('cfg2', '$v', $rep, round(d['ms_per_step'],2), round(g['ms_per_step'],2), round(g['edge_kernels']['fwd_ms_per_step'],2), round(g['edge_kernels']['bwd_ms_per_step'],2), round(g['e2e']['ms_per_step'],1))" >> gpurun_out/gat_ab8_ab.txt
  done
done
cat gpurun_out/gat_ab8_ab.txt
