# r2m: box topology (NUMA / CPU affinity of the GPU), e2e variance, phase marks, virtual-fleet batches sweep
set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r2m_topo.txt 2>&1; cat gpurun_out/r2m_topo.txt
lscpu | head -30 > gpurun_out/r2m_lscpu.txt; cat gpurun_out/r2m_lscpu.txt | grep -i "numa\|socket\|model name\|^CPU(s)"
cat /sys/bus/pci/devices/$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | tr 'A-Z' 'a-z' | sed 's/^0000//;s/^/0000/' | cut -c1-12)/numa_node 2>&1
nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader
free -g | head -2
timeout 600 python profiles/tools/var_diag.py > gpurun_out/r2m_phases.txt 2>&1; echo "phases rc=$?"; head -14 gpurun_out/r2m_phases.txt
for i in 1 2; do timeout 900 python bench.py --no-gat --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2m_bench_$i.json 2> gpurun_out/r2m_bench_$i.err; python -c "
import json; d=json.load(open('gpurun_out/r2m_bench_$i.json')); print('run $i', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],1), round(d['e2e_lean']['ms_per_step'],1), round(d['e2e_host_checkpoints']['ms_per_step'],1), round(d['e2e_hbm_budget']['ms_per_step'],1), round(d['virtual_fleet_m8']['ms_per_step'],1))"; done
timeout 1500 python profiles/tools/virt_sweep.py > gpurun_out/r2m_virt.txt 2>&1; echo "virt rc=$?"; grep '^{' gpurun_out/r2m_virt.txt | cut -c1-300
