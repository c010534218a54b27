#!/bin/bash
# full GPU suite at the working tree, then bench lines (selection ms) at A and C
set -u
mkdir -p gpurun_out/suite
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/suite/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/suite/pytest.txt
tail -4 gpurun_out/suite/pytest.txt
for c in A C M; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/suite/$c.json 2>/dev/null
  python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'step', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'sel_ms', round(d['select_ms'],3), 'share', round(d['select_share'],4), 'mhz', d['clocks']['sm_mhz'])" gpurun_out/suite/$c.json "$c"
done
for c in C A; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/suite/launches_$c.csv python bench.py --config $c --profile --no-e2e --no-cpu --no-dense --steps 2 --warmup 1 > /dev/null 2>&1
  python tools/launches.py gpurun_out/suite/launches_$c.csv 2>&1 | grep baatt
done
