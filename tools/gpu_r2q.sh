#!/bin/bash
# r2q: sampler starts kernel (parity + bench), the N > 1 step through NCCL with one rank, ranges ncu.
OUT=gpurun_out
timeout 600 python -m pytest tests/test_sampler_gpu.py -q -m gpu -x --timeout 300 > $OUT/r2q_tests.log 2>&1; echo rc=$?; tail -2 $OUT/r2q_tests.log
timeout 300 python bench.py --mode sample --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/r2q_bench_sample.json 2>&1; tail -c 500 $OUT/r2q_bench_sample.json
SC_FORCE_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --steps 50 --warmup 5 --no-cpu-baseline > $OUT/r2q_bench_forced_dist.json 2> $OUT/r2q_bench_forced_dist.err; echo fd_rc=$?; tail -c 1500 $OUT/r2q_bench_forced_dist.json; tail -3 $OUT/r2q_bench_forced_dist.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ranges" -c 3 -o $OUT/prof_r2q_ranges -f python bench.py --mode ranges --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu -i $OUT/prof_r2q_ranges.ncu-rep --page raw --csv > $OUT/raw_r2q_ranges.csv 2>/dev/null
rm -f $OUT/prof_r2q_ranges.ncu-rep
