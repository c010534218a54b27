#!/bin/bash
# Round-2 head verification: GPU suite, smoke, bench lines (C default + A/M/V, random lists, reference arm),
# launch lists + per-config attention traffic, one full ncu capture of the attention kernel at C.
set -u
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
tail -2 $O/pytest_gpu.txt; tail -3 $O/smoke.txt
timeout 900 python bench.py > $O/bench_C.json 2> $O/bench_C.err
for c in A M V; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python bench.py --config C --random-lists --no-e2e --no-cpu --no-dense > $O/bench_C_random.json 2> $O/bench_C_random.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
for f in C A M V C_random ref; do python -c "import json,sys; d=json.load(open('$O/bench_$f.json')); r=d.get('roofline') or {}; print('$f', round(d['value'],3), d['unit'], 'attn', r.get('achieved'), 'frac', r.get('frac'), 'sel_share', d.get('select_share'), 'dense', d.get('dense_tflops'), 'sdpa', d.get('sdpa_tflops'), 'e2e', (d.get('e2e') or {}).get('value'), 'mhz', (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'))" 2>&1 | tail -1; done
args=()
for c in C A M; do
  timeout 1400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_$c.csv python bench.py --config $c --profile --no-e2e --no-cpu --no-dense --steps 2 --warmup 1 > $O/launches_$c.log 2>&1
  python tools/launches.py $O/launches_$c.csv > $O/launches_$c.txt 2>&1
  kn=$(tail -1 $O/launches_$c.log | python -c "import json,sys; print(json.loads(sys.stdin.read())['roofline']['kernel'])")
  args+=($c $kn $O/launches_$c.csv)
done
python tools/attn_traffic.py "${args[@]}" > $O/attn_traffic.txt 2>&1
grep -h "baatt\|attn" $O/launches_C.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_pp_kernel -c 1 -o $O/attn_C_full python bench.py --config C --profile --no-e2e --no-cpu --no-dense --steps 1 --warmup 0 > $O/attn_C_full.log 2>&1
ls -la $O/*.ncu-rep
