#!/bin/bash
# Head check: GPU suite, smoke, per-config bench lines (selection share), launch list at A.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
for c in C A M V; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_A.csv python bench.py --config A --profile --no-e2e --no-cpu --no-dense --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_A.csv > gpurun_out/launches_A.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/smoke.txt
for c in C A M V; do python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'sel_ms', round(d['select_ms'],3), 'share', round(d['select_share'],4), 'launches', d['gpu_launches'], 'dense', d.get('dense_tflops'), 'sdpa', d.get('sdpa_tflops'), 'mhz', d['clocks']['sm_mhz'])"; done
