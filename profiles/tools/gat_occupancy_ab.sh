# Same-box A/B of the GAT row passes' occupancy inside the full bench run
# (the GAT sub-line, after the GCN runs): default vs variants built with
#   python -m paper_2311_14898_b200.build --variant s1m5 HT_GAT_S1_MINB=5
#   python -m paper_2311_14898_b200.build --variant d8 HT_GAT_DST_MINB=8
#   python -m paper_2311_14898_b200.build --variant s1m5d8 HT_GAT_S1_MINB=5 HT_GAT_DST_MINB=8
mkdir -p gpurun_out
for rep in 1 2; do
  for v in default s1m5 d8 s1m5d8; do
    if [ $v = default ]; then lib=paper_2311_14898_b200/lib/libhongtu_b200.so; else lib=paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so; fi
    HT_LIB=$lib timeout 900 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/e_ab_${v}_$rep.json 2> /dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/e_ab_${v}_$rep.json').read().strip().splitlines()[-1]); g=d['gat']; print('$v', $rep, round(d['ms_per_step'],2), round(g['ms_per_step'],2), round(g['edge_kernels']['fwd_ms_per_step'],2), round(g['edge_kernels']['bwd_ms_per_step'],2), round(g['e2e']['ms_per_step'],1))" >> gpurun_out/gat_occ_ab.txt
  done
done
cat gpurun_out/gat_occ_ab.txt
