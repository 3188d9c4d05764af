#!/bin/bash
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
line() {
  local label="$1"; shift
  env "$@" > $OUT/q.json 2>$OUT/q.err
  python - "$OUT/q.json" "$label" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f"{sys.argv[2]:40s} {d['value']:.3e}/s kernel {r['kernel_ms']*1e3:7.1f} us dense_frac {r['dense_frac']:.3f} frac {r['frac']:.3f} step {d['ms_per_step']*1e3:7.1f} us {r['eval_kernel']} {d.get('phases_us')}")
except Exception as e: print(sys.argv[2], "FAILED", e, open(sys.argv[1].replace('.json','.err')).read()[-800:])
PY
}
B="timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e"
line "f32 default"                 $B
line "f32 EPL0 chunk 2000"         SC_EPL=0 SC_FORCE_CHUNK=2000 $B
line "f32 EPL0 chunk 4000"         SC_EPL=0 SC_FORCE_CHUNK=4000 $B
line "f32 EPL0 chunk 1008"         SC_EPL=0 SC_FORCE_CHUNK=1008 $B
line "app_choice"                  $B --order app_choice
line "multi_select"                $B --order multi_select
line "bf16 app_choice"             $B --order app_choice --dtype bf16
echo "--- N=2 on one GPU (gloo) ---"
SC_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rows 262144 2>&1 | tail -2 | cut -c1-600
echo "--- reference arm under torchrun N=2 ---"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 2>&1 | tail -2 | cut -c1-300
