timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "selection" 2>&1 | tail -2
for cfg in A M; do
  timeout 200 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$cfg',d['roofline']['kernel'],'attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'sel',round(d['select_ms'],3),'share',round(d['select_share'],4),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
done
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"radix_scatter_kernel|gather_stats|scores" -c 6 -o gpurun_out/sel_full_A python bench.py --config A --profile --steps 1 --warmup 0 --no-e2e --no-dense --no-cpu > gpurun_out/ncu_sel.log 2>&1; echo ncu $?; tail -3 gpurun_out/ncu_sel.log
