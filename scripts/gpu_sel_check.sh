#!/bin/bash
# Selection change check: selection parity tests, bench lines A/C/M (no dense), C selection launch list.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "selection or fullsize or topp or norm_order or deterministic or block_mass or deviation" > gpurun_out/pytest_sel.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sel.txt; tail -3 gpurun_out/pytest_sel.txt
summ() { python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'step', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'sel_ms', round(d['select_ms'],3), 'share', round(d['select_share'],4), 'mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$1" "$2" 2>&1 | tail -1; }
for c in ${CFGS:-A C M}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/selchk_${c}.json 2>/dev/null; summ gpurun_out/selchk_${c}.json "$c"
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/sel_launches_C4.csv python bench.py --config C --profile --no-e2e --no-cpu --no-dense --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/sel_launches_C4.csv 2>&1 | grep baatt
