#!/bin/bash
# r5h: launch list of the sampler step (per-kernel share of its 41 us).
OUT=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r5h_launches_sample.csv python bench.py --mode sample --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/r5h_launches_sample.csv')) if len(r)>10]
h=rows[0]; i=h.index('Kernel Name'); v=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[1:]:
    d[r[i][:60]].append(float(r[v].replace(',','')))
for k,x in d.items(): print(len(x), round(sum(x)/len(x)/1000,2), 'us', k)
PY
