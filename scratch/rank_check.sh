#!/bin/bash
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_rank.py -x -q > $OUT/pytest_rank.log 2>&1; echo "rc $?" >> $OUT/pytest_rank.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?" >> $OUT/smoke.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "rc $?" >> $OUT/bench_n2.err
