#!/bin/bash
# r4a: session re-entry check on HEAD: full GPU suite, smoke, the driver's bench line.
OUT=gpurun_out
TAG=r4a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > $OUT/${TAG}_pytest_gpu.log 2>&1; echo all_rc=$?; tail -3 $OUT/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo smoke_rc=$?; tail -1 $OUT/${TAG}_smoke.log
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo bench_rc=$?; tail -1 $OUT/${TAG}_bench.json | cut -c1-600
timeout 300 python bench.py --config 2 --order multi_select --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_multiselect.json 2>/dev/null; tail -1 $OUT/${TAG}_bench_multiselect.json | cut -c1-300
