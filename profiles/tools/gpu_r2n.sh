# r2n: probe - community-major order + column slices for the one-device transposed aggregation
set -x
mkdir -p gpurun_out
for cfgk in "0 0" "128 0" "0 16" "128 16" "128 8" "64 16" "128 32"; do
  set -- $cfgk
  HT_COL_SLICE_BWD=$1 timeout 600 python profiles/tools/locality_order_probe.py $2 > gpurun_out/r2n_s$1_k$2.txt 2>&1
  grep -E "epoch 5|digest|LDG" gpurun_out/r2n_s$1_k$2.txt
done
