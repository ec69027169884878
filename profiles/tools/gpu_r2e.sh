# r2e: full GPU suite, cfg2 bench line, per-GPU shares cfg3s / cfg4s / cfg5s, GAT reference arm
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; free -g | head -2
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2e_gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2e_gputest.log
timeout 1200 python bench.py > gpurun_out/r2e_bench_cfg2.json 2> gpurun_out/r2e_bench_cfg2.err; echo "cfg2 rc=$?"
for c in cfg5s cfg3s cfg4s; do
  timeout 1800 python bench.py --config $c --no-gat --steps 3 --warmup 3 > gpurun_out/r2e_bench_$c.json 2> gpurun_out/r2e_bench_$c.err; echo "$c rc=$?"; tail -3 gpurun_out/r2e_bench_$c.err
done
timeout 900 python bench.py --impl reference --config cfg5s --steps 3 --warmup 1 > gpurun_out/r2e_ref_cfg5s.json 2> gpurun_out/r2e_ref_cfg5s.err; echo "ref5 rc=$?"
