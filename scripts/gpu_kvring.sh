timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 200 -o timeout_method=thread -x 2>&1 | tail -2
for cfg in A C; do
for mode in "BA_ATTN_DEBUG=1" "BA_ATTN_DEBUG=1 BA_ATTN_SKIPLOAD=3" "BA_ATTN_DEBUG=0"; do
  env $mode timeout 200 python bench.py --config $cfg --steps 5 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$cfg $mode','attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'clk',d['clocks']['sm_mhz'],d['clocks']['reasons'])" 2>&1 | tail -1
done; done
