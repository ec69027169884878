set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f1_gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f1_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f1_smoke.log
timeout 1200 python bench.py > gpurun_out/f1_bench_cfg2.json 2> gpurun_out/f1_bench_cfg2.err; echo "cfg2 rc=$?"
for c in cfg5s cfg3s cfg4s; do timeout 2400 python bench.py --config $c --no-gat --steps 3 --warmup 3 > gpurun_out/f1_bench_$c.json 2> gpurun_out/f1_bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f1_reference_arm.json 2> gpurun_out/f1_reference_arm.err; echo "ref rc=$?"
