# r2f: compute-sanitizer memcheck / racecheck / synccheck over every layer-driver path
set -x
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check full --error-exitcode 9 python profiles/tools/sanitize_epoch.py > gpurun_out/r2f_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -12 gpurun_out/r2f_memcheck.log
timeout 2400 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python profiles/tools/sanitize_epoch.py > gpurun_out/r2f_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -12 gpurun_out/r2f_racecheck.log
timeout 1500 $CS --tool synccheck --error-exitcode 9 python profiles/tools/sanitize_epoch.py > gpurun_out/r2f_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -8 gpurun_out/r2f_synccheck.log
# rank mode: two processes sharing the GPU, both under memcheck
( timeout 1200 $CS --tool memcheck --error-exitcode 9 python profiles/tools/sanitize_epoch.py --rank 0 > gpurun_out/r2f_rank0_memcheck.log 2>&1; echo "rank0 rc=$?" ) &
( timeout 1200 $CS --tool memcheck --error-exitcode 9 python profiles/tools/sanitize_epoch.py --rank 1 > gpurun_out/r2f_rank1_memcheck.log 2>&1; echo "rank1 rc=$?" ) &
wait
tail -6 gpurun_out/r2f_rank0_memcheck.log gpurun_out/r2f_rank1_memcheck.log
