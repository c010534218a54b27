#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "selection or fullsize or topp or norm_order or deterministic" > gpurun_out/pytest_scores.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_scores.txt; tail -3 gpurun_out/pytest_scores.txt
summ() { python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'step', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'sel_ms', round(d['select_ms'],3), 'share', round(d['select_share'],4), 'mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$1" "$2" 2>&1 | tail -1; }
for c in A C M; do
  for r in 1 2; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/sc_wide_${c}_$r.json 2>/dev/null; summ gpurun_out/sc_wide_${c}_$r.json "wide $c"
    BA_SCORES_NARROW=1 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/sc_narrow_${c}_$r.json 2>/dev/null; summ gpurun_out/sc_narrow_${c}_$r.json "narrow $c"
  done
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/sel_launches_C3.csv python bench.py --config C --profile --no-e2e --no-cpu --no-dense --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/sel_launches_C3.csv 2>&1 | grep baatt
