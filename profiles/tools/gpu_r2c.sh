# r2c: TMA-store GEMM epilogue - unit/epoch parity, rates A/B, value A/B; PCIe counters (app-range)
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_epoch.py tests/test_gpu_gat.py tests/test_gpu_cache.py -x -q -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2c_tests.log
timeout 600 python profiles/tools/tf32_peak.py > gpurun_out/r2c_rates_tma.json 2>&1; echo "rates rc=$?"
HT_NO_TMA_STORE=1 timeout 600 python profiles/tools/tf32_peak.py > gpurun_out/r2c_rates_notma.json 2>&1
python - <<'PY'
import json
a=json.load(open("gpurun_out/r2c_rates_tma.json")); b=json.load(open("gpurun_out/r2c_rates_notma.json"))
for k in a:
    if isinstance(a[k], dict): print(f"{k:28s} tma {a[k]['ms']:.3f} ms  scalar {b[k]['ms']:.3f} ms")
PY
for v in 0 1; do
  HT_NO_TMA_STORE=$v timeout 600 python bench.py --only-value --no-gat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_ab_$v.log 2>&1
  grep "value run" gpurun_out/r2c_ab_$v.log
done
timeout 900 ncu --replay-mode app-range --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_pcie_e2e.csv python bench.py --profile-epoch e2e --steps 1 --warmup 2 > gpurun_out/r2c_pcie_e2e.log 2>&1; echo "pcie e2e rc=$?"; tail -8 gpurun_out/r2c_pcie_e2e.csv; tail -3 gpurun_out/r2c_pcie_e2e.log
timeout 900 ncu --replay-mode app-range --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_pcie_virt.csv python bench.py --profile-epoch virt --steps 1 --warmup 1 > gpurun_out/r2c_pcie_virt.log 2>&1; echo "pcie virt rc=$?"; tail -8 gpurun_out/r2c_pcie_virt.csv; tail -3 gpurun_out/r2c_pcie_virt.log
