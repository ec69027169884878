# r2l: full GPU suite + cfg2 bench line + cfg5s line + phase marks (after the r2 kernel changes)
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2l_gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2l_gputest.log
timeout 1200 python bench.py > gpurun_out/r2l_bench_cfg2.json 2> gpurun_out/r2l_bench_cfg2.err; echo "cfg2 rc=$?"
timeout 1800 python bench.py --config cfg5s --no-gat --steps 3 --warmup 3 > gpurun_out/r2l_bench_cfg5s.json 2> gpurun_out/r2l_bench_cfg5s.err; echo "cfg5s rc=$?"
timeout 600 python profiles/tools/var_diag.py > gpurun_out/r2l_phases.txt 2>&1; echo "phases rc=$?"; head -14 gpurun_out/r2l_phases.txt
