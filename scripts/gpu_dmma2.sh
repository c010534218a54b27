timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "selection or topp" 2>&1 | tail -2
for cfg in M C A; do
for mode in "" "BA_SCORES_SIMT=1"; do
  env $mode timeout 200 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$cfg $mode','attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'sel',round(d['select_ms'],3),'share',round(d['select_share'],4),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
  tail -1 gpurun_out/p.err
done; done
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active --clock-control none -k regex:"scores" -c 2 --csv python bench.py --config M --profile --steps 1 --warmup 0 --no-e2e --no-dense --no-cpu 2>/dev/null | grep -v "^==" | cut -c1-200 | tail -8
