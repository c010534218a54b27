#!/bin/bash
# pair-kernel variants by BA_LIB_PATH: parity subset, then bench lines at A, C, C random lists
#   bash scripts/gpu_variants.sh "base p1 se p1se"   (base = libbaatt.so, X = libbaatt_X.so)
set -u
mkdir -p gpurun_out/var
V=$1; CFG=${2:-"A C Crand"}
lib() { [ "$1" = base ] && echo paper_2605_19726_b200/libbaatt.so || echo paper_2605_19726_b200/libbaatt_$1.so; }
for v in $V; do
  BA_LIB_PATH=$(lib $v) timeout 900 python -m pytest tests -m gpu -q -x -k "dissimilar or split_steps or b128 or smoke or determinism" > gpurun_out/var/pytest_$v.txt 2>&1
  echo "$v pytest: $(tail -1 gpurun_out/var/pytest_$v.txt)"
done
for r in 1 2; do
  for c in $CFG; do
    for v in $V; do
      extra=""; cc=$c
      [ "$c" = Crand ] && { extra="--random-lists"; cc=C; }
      BA_LIB_PATH=$(lib $v) timeout 600 python bench.py --config $cc $extra --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/var/${v}_${c}_$r.json 2>/dev/null
      python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'step', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'mhz', d['clocks']['sm_mhz'])" gpurun_out/var/${v}_${c}_$r.json "$v $c" 2>&1 | tail -1
    done
  done
done
