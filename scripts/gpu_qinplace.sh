#!/bin/bash
# Q read in place by the softmax warps (no Q' copy): parity + A/B vs the copies at A, C, V
set -u
mkdir -p gpurun_out/qip
timeout 900 python -m pytest tests -m gpu -q -x -k "zero_copy or gather or smoke" > gpurun_out/qip/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/qip/pytest.txt
tail -3 gpurun_out/qip/pytest.txt
summ() { python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'step', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'sel_ms', round(d['select_ms'],3), 'share', round(d['select_share'],4), 'mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$1" "$2" 2>&1 | tail -1; }
for c in A C V; do
  for r in 1 2; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense --q-in-place > gpurun_out/qip/${c}_qip_$r.json 2>/dev/null; summ gpurun_out/qip/${c}_qip_$r.json "q-in-place $c"
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/qip/${c}_copy_$r.json 2>/dev/null; summ gpurun_out/qip/${c}_copy_$r.json "copies     $c"
  done
done
