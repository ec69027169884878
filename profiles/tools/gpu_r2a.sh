set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2a_gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2a_gputest.log
timeout 900 python bench.py > gpurun_out/r2a_bench.log 2>gpurun_out/r2a_bench.err; echo "bench rc=$?"
tail -2 gpurun_out/r2a_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2a_ref.log 2>gpurun_out/r2a_ref.err; echo "ref rc=$?"
tail -2 gpurun_out/r2a_ref.log
