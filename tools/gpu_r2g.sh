#!/bin/bash
# r2g: dense-mapped eval path (column-compacted rows): parity + cfg3-compact / cfg2-compact bench + ncu.
OUT=gpurun_out
timeout 900 python -m pytest tests/test_compact_gpu.py tests/test_parity_gpu.py -q -m gpu -x --timeout 300 > $OUT/r2g_tests.log 2>&1; echo tests_rc=$?
tail -15 $OUT/r2g_tests.log
for cfg in "3 f32" "3 bf16" "2 f32"; do set -- $cfg
  for dm in 1 0; do
    SC_DM=$dm timeout 600 python bench.py --config $1 --dtype $2 --compact --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2g_c$1_$2_dm$dm.json 2>&1
    echo "cfg$1 $2 compact dm=$dm: $(python -c "import json;d=json.loads(open('$OUT/r2g_c$1_$2_dm$dm.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['eval_kernel'],round(r['kernel_ms'],4),round(r['frac'],3), round(d['value']/1e9,3),'G/s')")"
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" -s 3 -c 1 -o $OUT/prof_r2g_cfg3c -f python bench.py --config 3 --compact --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu -i $OUT/prof_r2g_cfg3c.ncu-rep --page raw --csv > $OUT/raw_r2g_cfg3c.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r2g_launches_cfg3c.csv python bench.py --config 3 --compact --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py $OUT/prof_r2g_cfg3c.ncu-rep $OUT/r2g_launches_cfg3c.csv $OUT/ncu_eval_cfg3_compact_f32.json $OUT/r2g_eval_cfg3_compact_f32.txt 524288 eval_kernel > /dev/null 2>&1
rm -f $OUT/prof_r2g_cfg3c.ncu-rep
