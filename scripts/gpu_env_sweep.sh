#!/bin/bash
# Env-knob sweep: gpurun -- bash scripts/gpu_env_sweep.sh CFG "ENV1" "ENV2" ...   ("-" = no env)
set -u
mkdir -p gpurun_out
CFG=$1; shift
summ() { python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'step', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'sel_ms', round(d['select_ms'],3), 'mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$1" "$2" 2>&1 | tail -1; }
for r in 1 2; do
  for e in "$@"; do
    tag=$(echo "$e" | tr -c 'A-Za-z0-9' '_')
    if [ "$e" = "-" ]; then timeout 600 python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/es_${CFG}_${tag}_$r.json 2>/dev/null
    else env $e timeout 600 python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/es_${CFG}_${tag}_$r.json 2>/dev/null; fi
    summ gpurun_out/es_${CFG}_${tag}_$r.json "$CFG [$e] r$r"
  done
done
