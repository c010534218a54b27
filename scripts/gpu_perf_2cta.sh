for cfg in C A V; do
for mode in "BA_ATTN_1CTA=1" "BA_ATTN_1CTA=0"; do
  env $mode timeout 200 python bench.py --config $cfg --steps 5 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$cfg $mode','attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'sel',round(d['select_ms'],2),'clk',d['clocks']['sm_mhz'],d['clocks']['reasons'])"
done; done
