#!/bin/bash
# r2t: compute-sanitizer on every kernel family incl. the round-2 kernels.
OUT=gpurun_out
timeout 600 python tools/sanitize_kernels.py > $OUT/r2t_plain.log 2>&1; echo plain_rc=$?; tail -3 $OUT/r2t_plain.log
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_kernels.py > $OUT/r2t_sanitizer_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 $OUT/r2t_sanitizer_$tool.log
done
