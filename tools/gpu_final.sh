#!/bin/bash
# Round-end evidence: bench line (default config) + reference arm + ncu launch list + ncu full
# captures (eval f32 / bf16, head) + the N = 2 bench path on one GPU (gloo) + head bench.
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r1}
mkdir -p $OUT
nproc; lscpu | grep "Model name"
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; tail -1 $OUT/pytest_gpu_$TAG.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > $OUT/clocks_$TAG.csv &
SMI=$!
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
kill $SMI
tail -1 $OUT/bench_$TAG.json | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
tail -1 $OUT/bench_ref_$TAG.json | cut -c1-200
timeout 600 python bench.py --mode head --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench_head_$TAG.json 2>/dev/null
tail -1 $OUT/bench_head_$TAG.json | cut -c1-200
timeout 300 python bench.py --mode ranges --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench_ranges_$TAG.json 2>/dev/null
timeout 300 python bench.py --mode sample --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench_sample_$TAG.json 2>/dev/null
timeout 600 python bench.py --mode all_apps --config 4 --rows 1048576 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/bench_allapps_$TAG.json 2>/dev/null
timeout 300 python bench.py --config 4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench_cfg4_$TAG.json 2>/dev/null
timeout 300 python bench.py --config 2 --order app_choice --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench_appchoice_$TAG.json 2>/dev/null
tail -qn1 $OUT/bench_ranges_$TAG.json $OUT/bench_sample_$TAG.json $OUT/bench_allapps_$TAG.json $OUT/bench_cfg4_$TAG.json $OUT/bench_appchoice_$TAG.json | cut -c1-160
SC_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_n2share_$TAG.json 2> $OUT/bench_n2share_$TAG.err
tail -1 $OUT/bench_n2share_$TAG.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" -s 3 -c 1 \
    -o $OUT/prof_${TAG}_f32 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" -s 3 -c 1 \
    -o $OUT/prof_${TAG}_bf16 -f python bench.py --dtype bf16 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"head_kernel" -s 2 -c 1 \
    -o $OUT/prof_${TAG}_head -f python bench.py --mode head --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hist" -s 3 -c 1 \
    -o $OUT/prof_${TAG}_hist -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls $OUT/*.ncu-rep
# summaries on the box (the .ncu-rep files of the eval kernel are ~30 MB each: over gpurun's 64 MiB)
python tools/ncu_summary.py $OUT/prof_${TAG}_f32.ncu-rep $OUT/launches_$TAG.csv $OUT/ncu_eval_cfg2_f32.json $OUT/${TAG}_eval_cfg2_f32.txt 1048576 eval_kernel > /dev/null
python tools/ncu_summary.py $OUT/prof_${TAG}_bf16.ncu-rep $OUT/launches_$TAG.csv $OUT/ncu_eval_cfg2_bf16.json $OUT/${TAG}_eval_cfg2_bf16.txt 1048576 eval_kernel > /dev/null
python tools/ncu_summary.py $OUT/prof_${TAG}_head.ncu-rep $OUT/launches_$TAG.csv $OUT/ncu_head_cfg2_d2048.json $OUT/${TAG}_head_cfg2_d2048.txt 1048576 head_kernel > /dev/null
python tools/ncu_summary.py $OUT/prof_${TAG}_hist.ncu-rep $OUT/launches_$TAG.csv $OUT/ncu_hist_cfg2.json $OUT/${TAG}_hist_cfg2.txt 1048576 hist > /dev/null
ncu -i $OUT/prof_${TAG}_bf16.ncu-rep --page source --csv --print-source sass > $OUT/src_${TAG}_bf16.csv 2>/dev/null
ncu -i $OUT/prof_${TAG}_f32.ncu-rep --page raw --csv > $OUT/raw_${TAG}_f32.csv 2>/dev/null
ncu -i $OUT/prof_${TAG}_head.ncu-rep --page raw --csv > $OUT/raw_${TAG}_head.csv 2>/dev/null
rm -f $OUT/prof_${TAG}_f32.ncu-rep $OUT/prof_${TAG}_bf16.ncu-rep $OUT/prof_${TAG}_hist.ncu-rep
du -sh $OUT
