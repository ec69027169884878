# The round's measurement commands on one B200 (run from the repo root under
# gpurun; outputs in gpurun_out/, summaries copied to profiles/ by hand).
set -x
mkdir -p gpurun_out
# 1. parity: the GPU suite, the driver's smoke
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()"
# 2. contract lines: cfg 2 (default), the per-GPU shares, the CPU reference arm
timeout 1200 python bench.py > gpurun_out/bench_cfg2.json
for c in cfg3s cfg4s cfg5s; do
  timeout 2400 python bench.py --config $c --no-gat --steps 3 --warmup 3 > gpurun_out/bench_$c.json
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/reference_arm.json
# 3. launch lists of one profiled epoch (cudaProfilerStart/Stop around it) -> profiles/r2_*launches*, r2_traffic.json
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none --csv --log-file gpurun_out/value_launches.csv python bench.py --profile-epoch value --steps 1 --warmup 2
python profiles/summarize_launches.py gpurun_out/value_launches.csv > gpurun_out/value_launches.txt
python profiles/make_traffic.py gpurun_out/value_launches.csv 1 > gpurun_out/traffic.json
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/gat_launches.csv python bench.py --profile-epoch value --kind gat --steps 1 --warmup 2
# 4. full captures of the top kernels -> profiles/r2_ncu_*.txt (profiles/summarize_ncu.py)
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_seg_work_v4 -c 1 \
    -o gpurun_out/seg_work python bench.py --profile-epoch value --steps 1 --warmup 2
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_tc_gemm -c 2 \
    -o gpurun_out/tc_gemm python bench.py --profile-epoch value --steps 1 --warmup 2
# 5. PCIe counters of whole epochs -> profiles/r2_pcie_counters.json (profiles/tools/pcie_counters.py)
ncu --replay-mode app-range --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/pcie_e2e.csv python bench.py --profile-epoch e2e --steps 1 --warmup 2 > gpurun_out/pcie_e2e.log
ncu --replay-mode app-range --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/pcie_virt.csv python bench.py --profile-epoch virt --steps 1 --warmup 1 > gpurun_out/pcie_virt.log
# 6. TF32 ceiling and the path's GEMM rates; per-layer phase times; the virtual-fleet batch sweep
python profiles/tools/tf32_peak.py > gpurun_out/tf32_rates.json
python profiles/tools/var_diag.py > gpurun_out/phases.txt
python profiles/tools/virt_sweep.py > gpurun_out/virt_sweep.txt
# 7. compute-sanitizer over every layer-driver path (single process, then two ranks sharing the GPU)
CS=/usr/local/cuda/bin/compute-sanitizer
$CS --tool memcheck --leak-check full --error-exitcode 9 python profiles/tools/sanitize_epoch.py > gpurun_out/memcheck.log 2>&1
$CS --tool racecheck --racecheck-report all --error-exitcode 9 python profiles/tools/sanitize_epoch.py > gpurun_out/racecheck.log 2>&1
$CS --tool synccheck --error-exitcode 9 python profiles/tools/sanitize_epoch.py > gpurun_out/synccheck.log 2>&1
( $CS --tool memcheck --error-exitcode 9 python profiles/tools/sanitize_epoch.py --rank 0 > gpurun_out/rank0_memcheck.log 2>&1 ) &
( $CS --tool memcheck --error-exitcode 9 python profiles/tools/sanitize_epoch.py --rank 1 > gpurun_out/rank1_memcheck.log 2>&1 ) &
wait
# 8. full-size graphs with the streaming generator (host side)
python profiles/tools/synth_scale.py cfg5
python profiles/tools/synth_scale.py cfg3
