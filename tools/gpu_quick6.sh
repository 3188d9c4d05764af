#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
SC_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline --rows 262144 > $OUT/n2.log 2>&1
grep -E "Error|error|Traceback|^\{" $OUT/n2.log | head -20 | cut -c1-400
