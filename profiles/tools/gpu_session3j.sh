# Last check of session 3: the GPU suite and smoke with the final build.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/m_gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/m_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/m_smoke.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/m_bench_cfg2.json 2> gpurun_out/m_bench_cfg2.err; echo "cfg2 rc=$?"
