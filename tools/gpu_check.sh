#!/bin/bash
# Re-entry check: smoke, every GPU parity test, one default bench line.
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
nvidia-smi > $OUT/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -2 $OUT/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; tail -15 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -1 $OUT/bench.json
