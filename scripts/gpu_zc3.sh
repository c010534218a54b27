timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -x 2>&1 | tail -3
for cfg in A C M V; do
for mode in "" "--copies"; do
  timeout 200 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense $mode > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$cfg $mode',d['roofline']['kernel'],'zc',d['config']['zero_copy'],'attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'sel',round(d['select_ms'],3),'share',round(d['select_share'],4),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
  tail -1 gpurun_out/p.err
done; done
