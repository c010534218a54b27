#!/bin/bash
# A/B of two builds of libbaatt (product vs BA_LIB_PATH=$1) on bench configs; optional pytest first.
#   gpurun -- bash scripts/gpu_ab.sh paper_2605_19726_b200/libbaatt_X.so "A C" [pytest-k-expr|all|none] [extra bench flags]
set -u
mkdir -p gpurun_out
ALT=$1; CFGS=$2; K=${3:-none}; EXTRA=${4:-}
if [ "$K" = "all" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
elif [ "$K" != "none" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
fi
[ "$K" != "none" ] && tail -15 gpurun_out/pytest_gpu.txt
summ() { python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'step', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'sel_ms', round(d['select_ms'],3), 'share', round(d['select_share'],4), 'dense', d.get('dense_tflops'), 'sdpa', d.get('sdpa_tflops'), 'mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$1" "$2" 2>&1 | tail -1; }
for c in $CFGS; do
  for r in 1 2; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu $EXTRA > gpurun_out/ab_new_${c}${EXTRA// /}_$r.json 2> gpurun_out/ab_new_${c}${EXTRA// /}_$r.err
    summ gpurun_out/ab_new_${c}${EXTRA// /}_$r.json "new $c $EXTRA"
    BA_LIB_PATH=$ALT timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu $EXTRA > gpurun_out/ab_alt_${c}${EXTRA// /}_$r.json 2> gpurun_out/ab_alt_${c}${EXTRA// /}_$r.err
    summ gpurun_out/ab_alt_${c}${EXTRA// /}_$r.json "alt $c $EXTRA"
  done
done
