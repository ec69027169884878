#!/bin/bash
# N>1 bench path (rank mode, CUDA IPC, device-side barriers) with two
# processes sharing the box's one GPU
OUT=gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-gat > $OUT/bench2.json 2> $OUT/bench2.err; echo "rc $?" >> $OUT/bench2.err
