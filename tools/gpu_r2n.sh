#!/bin/bash
# r2n: lane-per-application all-apps kernel (parity, bench vs the warp kernel), head with
# shared-space bias loads (parity, bench, trace).
OUT=gpurun_out
timeout 900 python -m pytest tests/test_allapps_gpu.py -q -m gpu -x --timeout 300 > $OUT/r2n_allapps_tests.log 2>&1; echo aa_rc=$?; tail -5 $OUT/r2n_allapps_tests.log
for m in "SC_NOP=1" "SC_ALLAPPS=warp"; do
  env $m timeout 600 python bench.py --mode all_apps --config 4 --rows 1048576 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/r2n_allapps.json 2>&1
  echo "all-apps [$m]: $(python -c "import json;d=json.loads(open('$OUT/r2n_allapps.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3),'ms', '%.3g'%d['value'], d['roofline']['frac'])")"
done
cp $OUT/r2n_allapps.json $OUT/r2n_allapps_warp.json
timeout 600 python bench.py --mode all_apps --config 4 --rows 1048576 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/r2n_allapps.json 2>&1
timeout 900 python -m pytest tests/test_head_gpu.py -q -m gpu -x --timeout 240 > $OUT/r2n_head_tests.log 2>&1; echo head_rc=$?; tail -3 $OUT/r2n_head_tests.log
rm -f /tmp/trace.bin
SC_HEAD_TRACE=/tmp/trace.bin timeout 300 python bench.py --mode head --d 2048 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/head_trace.py /tmp/trace.bin 2>&1 | tail -2
timeout 300 python bench.py --mode head --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/r2n_head.json 2>&1
echo "head cfg2: $(python -c "import json;d=json.loads(open('$OUT/r2n_head.json').read().strip().splitlines()[-1]);r=d['roofline'];print(r['kernel'],round(r['kernel_ms'],4),round(r['frac'],3))")"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"all_apps" -s 1 -c 1 -o $OUT/prof_r2n_allapps -f python bench.py --mode all_apps --config 4 --rows 262144 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r2n_launches_allapps.csv python bench.py --mode all_apps --config 4 --rows 262144 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py $OUT/prof_r2n_allapps.ncu-rep $OUT/r2n_launches_allapps.csv $OUT/ncu_allapps_lane_cfg4.json $OUT/r2n_allapps_lane_cfg4.txt 262144 all_apps > /dev/null 2>&1
ncu -i $OUT/prof_r2n_allapps.ncu-rep --page raw --csv > $OUT/raw_r2n_allapps.csv 2>/dev/null
rm -f $OUT/prof_r2n_allapps.ncu-rep
