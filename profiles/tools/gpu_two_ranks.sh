set -x
mkdir -p gpurun_out
# two ranks (torchrun) sharing the one GPU: the multi-GPU code path of bench.py end to end
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --no-gat --no-cpu-baseline > gpurun_out/r2w_2ranks.json 2> gpurun_out/r2w_2ranks.err; echo "2ranks rc=$?"; tail -c 600 gpurun_out/r2w_2ranks.json; grep -i "error\|Traceback" gpurun_out/r2w_2ranks.err | head -5
