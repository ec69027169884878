# r2h: launch list of the current code (traffic), ncu --set full of the top kernel, GAT A/B
set -x
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r2h_value_launches.csv python bench.py --profile-epoch value --steps 1 --warmup 2 > gpurun_out/r2h_ncu_value.log 2>&1; echo "ncu rc=$?"
python profiles/summarize_launches.py gpurun_out/r2h_value_launches.csv > gpurun_out/r2h_value_launches.txt 2>&1; head -24 gpurun_out/r2h_value_launches.txt
python profiles/make_traffic.py gpurun_out/r2h_value_launches.csv 1 > gpurun_out/r2h_traffic.json; cat gpurun_out/r2h_traffic.json
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_seg_work_v4 -c 1 -o gpurun_out/r2h_seg_work python bench.py --profile-epoch value --steps 1 --warmup 2 > gpurun_out/r2h_ncu_full.log 2>&1; echo "full rc=$?"
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_tc_gemm -c 2 -o gpurun_out/r2h_tc_gemm python bench.py --profile-epoch value --steps 1 --warmup 2 > gpurun_out/r2h_ncu_full_gemm.log 2>&1; echo "full gemm rc=$?"
for v in default gat_du8 gat_su16; do
  if [ $v = default ]; then L=""; else L="paper_2311_14898_b200/lib/variants/$v/libhongtu_b200.so"; fi
  HT_LIB=$L timeout 900 python bench.py --only-value --kind gat --steps 5 --warmup 3 > gpurun_out/r2h_gat_$v.log 2>&1
  python - $v <<'PY'
import json,sys
for l in open(f"gpurun_out/r2h_gat_{sys.argv[1]}.log"):
    if "GAT:" in l:
        d=json.loads(l.split("GAT: ",1)[1]); print(sys.argv[1], round(d["ms_per_step"],2), d["edge_kernels"]["fwd_ms_per_step"], d["edge_kernels"]["bwd_ms_per_step"])
PY
done
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python profiles/tools/sanitize_epoch.py > gpurun_out/r2h_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/r2h_memcheck.log
timeout 2400 python bench.py --config cfg4s --no-gat --steps 3 --warmup 3 > gpurun_out/r2h_bench_cfg4s.json 2> gpurun_out/r2h_bench_cfg4s.err; echo "cfg4s rc=$?"; grep "^\[bench\]" gpurun_out/r2h_bench_cfg4s.err; tail -2 gpurun_out/r2h_bench_cfg4s.err
