#!/bin/bash
# r4f: all-apps lane kernel with one arg max per (row, application) instead of split maxima.
OUT=gpurun_out
TAG=${TAG:-r4f}
timeout 900 python -m pytest tests/test_allapps_gpu.py -q -m gpu --timeout 600 > $OUT/${TAG}_pytest.log 2>&1; echo rc=$?; tail -2 $OUT/${TAG}_pytest.log
timeout 600 python bench.py --mode all_apps --config 4 --rows 1048576 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_allapps.json 2>/dev/null
timeout 600 python bench.py --mode all_apps --config 4 --rows 1048576 --dtype bf16 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_allapps_bf16.json 2>/dev/null
for f in $OUT/${TAG}_bench_*.json; do tail -1 $f | cut -c1-700; echo; done
