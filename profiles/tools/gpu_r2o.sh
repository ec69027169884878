# r2o: full-size graphs with the streaming generator (host side only)
set -x
mkdir -p gpurun_out
free -g | head -2; nproc; df -h /tmp | tail -1
timeout 1500 python profiles/tools/synth_scale.py cfg5 > gpurun_out/r2o_cfg5.json 2> gpurun_out/r2o_cfg5.err; echo "cfg5 rc=$?"; cat gpurun_out/r2o_cfg5.json; tail -2 gpurun_out/r2o_cfg5.err
avail=$(awk '/MemAvailable/ {print int($2/1e6)}' /proc/meminfo)
if [ "$avail" -gt 120 ]; then
  timeout 2400 python profiles/tools/synth_scale.py cfg3 > gpurun_out/r2o_cfg3.json 2> gpurun_out/r2o_cfg3.err; echo "cfg3 rc=$?"; cat gpurun_out/r2o_cfg3.json; tail -2 gpurun_out/r2o_cfg3.err
fi
