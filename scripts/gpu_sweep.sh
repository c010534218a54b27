#!/bin/bash
# Sweep A/B library builds: gpurun -- bash scripts/gpu_sweep.sh "CFGS" "EXTRA" lib1.so lib2.so ...  (product lib = "prod")
set -u
mkdir -p gpurun_out
CFGS=$1; EXTRA=$2; shift 2
summ() { python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'step', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'sel_ms', round(d['select_ms'],3), 'dense', d.get('dense_tflops'), 'sdpa', d.get('sdpa_tflops'), 'mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$1" "$2" 2>&1 | tail -1; }
for r in 1 2; do
  for c in $CFGS; do
    for lib in "$@"; do
      tag=$(basename $lib .so)
      if [ "$lib" = "prod" ]; then
        timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu $EXTRA > gpurun_out/sw_${tag}_${c}_$r.json 2> gpurun_out/sw_${tag}_${c}_$r.err
      else
        BA_LIB_PATH=$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu $EXTRA > gpurun_out/sw_${tag}_${c}_$r.json 2> gpurun_out/sw_${tag}_${c}_$r.err
      fi
      summ gpurun_out/sw_${tag}_${c}_$r.json "$tag $c r$r"
    done
  done
done
