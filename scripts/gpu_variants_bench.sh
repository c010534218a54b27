#!/bin/bash
# bench-only variants (timing experiments that are not correct programs): A and C, 2 repeats
set -u
mkdir -p gpurun_out/var
V=$1; CFG=${2:-"A C"}
lib() { [ "$1" = base ] && echo paper_2605_19726_b200/libbaatt.so || echo paper_2605_19726_b200/libbaatt_$1.so; }
for r in 1 2; do for c in $CFG; do for v in $V; do
  BA_LIB_PATH=$(lib $v) timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/var/${v}_${c}_$r.json 2>/dev/null
  python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'step', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'mhz', d['clocks']['sm_mhz'])" gpurun_out/var/${v}_${c}_$r.json "$v $c" 2>&1 | tail -1
done; done; done
