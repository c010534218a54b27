#!/bin/bash
# pp64 check: targeted GPU tests, then M bench with the B = 64 pair kernel vs the dual-tile kernel, A selection launches.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "b64 or dissimilar or running_max or unequal or selection or fullsize or attention_bf16_B64 or deterministic or units" > gpurun_out/pytest_pp64.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pp64.txt
tail -15 gpurun_out/pytest_pp64.txt
summ() { python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'step', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'kernel', d['roofline']['kernel'], 'sel_ms', round(d['select_ms'],3), 'share', round(d['select_share'],4), 'dense', d.get('dense_tflops'), 'sdpa', d.get('sdpa_tflops'), 'mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$1" "$2" 2>&1 | tail -1; }
for r in 1 2; do
  BA_ATTN_B64=pp timeout 600 python bench.py --config M --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/m_pp_$r.json 2> gpurun_out/m_pp_$r.err; summ gpurun_out/m_pp_$r.json "pp64 M"
  timeout 600 python bench.py --config M --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/m_dual_$r.json 2> gpurun_out/m_dual_$r.err; summ gpurun_out/m_dual_$r.json "dual M"
done
BA_ATTN_B64=pp timeout 600 python bench.py --config M --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense --random-lists > gpurun_out/m_pp_rand.json 2> gpurun_out/m_pp_rand.err; summ gpurun_out/m_pp_rand.json "pp64 M random"
timeout 600 python bench.py --config M --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense --random-lists > gpurun_out/m_dual_rand.json 2> gpurun_out/m_dual_rand.err; summ gpurun_out/m_dual_rand.json "dual M random"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/sel_launches_A2.csv python bench.py --config A --profile --no-e2e --no-cpu --no-dense --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/sel_launches_A2.csv 2>&1 | grep baatt
