#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
bash tools/gpu_final.sh
