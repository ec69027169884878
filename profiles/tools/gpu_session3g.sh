# Session-3 final check on one B200: GPU suite, smoke, the contract lines
# (cfg 2 incl. the GAT sub-line, cfg5s GAT share), launch lists of one
# GCN and one GAT value epoch.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g_gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/g_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g_smoke.log
timeout 1200 python bench.py > gpurun_out/g_bench_cfg2.json 2> gpurun_out/g_bench_cfg2.err; echo "cfg2 rc=$?"
timeout 2400 python bench.py --config cfg5s --no-gat --steps 3 --warmup 3 > gpurun_out/g_bench_cfg5s.json 2> gpurun_out/g_bench_cfg5s.err; echo "cfg5s rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none --csv --log-file gpurun_out/g_value_launches.csv python bench.py --profile-epoch value --steps 1 --warmup 2 > gpurun_out/g_ncu_list.log 2>&1; echo "ncu rc=$?"
python profiles/summarize_launches.py gpurun_out/g_value_launches.csv > gpurun_out/g_value_launches.txt
python profiles/make_traffic.py gpurun_out/g_value_launches.csv 1 > gpurun_out/g_traffic.json
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/g_gat_launches.csv python bench.py --profile-epoch value --kind gat --steps 1 --warmup 2 > gpurun_out/g_ncu_gat.log 2>&1; echo "ncu gat rc=$?"
python profiles/summarize_launches.py gpurun_out/g_gat_launches.csv > gpurun_out/g_gat_launches.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g_reference_arm.json 2> gpurun_out/g_reference_arm.err; echo "ref rc=$?"
