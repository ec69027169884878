# compute-sanitizer over every layer-driver path incl. the session-3 GEMMs
# (CTA-pair 3xTF32, masked-A backward) -> profiles/sanitizer/r3_*.log
set -x
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check full --error-exitcode 9 python profiles/tools/sanitize_epoch.py > gpurun_out/r3_memcheck_leakcheck.log 2>&1; echo "memcheck rc=$?"
timeout 1500 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python profiles/tools/sanitize_epoch.py > gpurun_out/r3_racecheck.log 2>&1; echo "racecheck rc=$?"
timeout 1500 $CS --tool synccheck --error-exitcode 9 python profiles/tools/sanitize_epoch.py > gpurun_out/r3_synccheck.log 2>&1; echo "synccheck rc=$?"
tail -2 gpurun_out/r3_*.log
