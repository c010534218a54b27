#!/bin/bash
# Evidence at head: attention-kernel DRAM traffic per config (launch lists -> profiles/attn_traffic.json),
# one ncu --set full capture of the attention kernel at C, and cuDNN SDPA vs ours (dense, A shapes) with source.
set -u
mkdir -p gpurun_out
args=()
for c in C A V M; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$c.csv python bench.py --config $c --profile --no-e2e --no-cpu --no-dense --steps 2 --warmup 1 > gpurun_out/launches_$c.log 2>&1
  python tools/launches.py gpurun_out/launches_$c.csv > gpurun_out/launches_$c.txt 2>&1
  kn=$(python -c "import json; print(json.load(open('gpurun_out/launches_$c.log'))['roofline']['kernel'])" 2>/dev/null || tail -1 gpurun_out/launches_$c.log | python -c "import json,sys; print(json.loads(sys.stdin.read())['roofline']['kernel'])")
  args+=($c $kn gpurun_out/launches_$c.csv)
done
python tools/attn_traffic.py "${args[@]}" > gpurun_out/attn_traffic.txt 2>&1; cat gpurun_out/attn_traffic.txt | head -40
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_pp_kernel -c 1 -o gpurun_out/attn_C_full python bench.py --config C --profile --no-e2e --no-cpu --no-dense --steps 1 --warmup 0 > gpurun_out/attn_C_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sdpa|attn_pp_kernel" -c 2 -o gpurun_out/sdpa_vs_ours python tools/sdpa_prof.py > gpurun_out/sdpa_vs_ours.log 2>&1
ls -la gpurun_out/*.ncu-rep
