#!/bin/bash
# r2d: full GPU suite + smoke + default bench on the committed round-2 code (libsc.so built here, shipped in-tree).
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu > $OUT/r2d_pytest_gpu.log 2>&1; echo all_rc=$?
tail -30 $OUT/r2d_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r2d_smoke.log 2>&1; echo smoke_rc=$?; tail -3 $OUT/r2d_smoke.log
timeout 600 python bench.py --steps 100 --warmup 10 > $OUT/r2d_bench.json 2> $OUT/r2d_bench.err; echo bench_rc=$?
tail -c 2500 $OUT/r2d_bench.json
