timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider --timeout 200 -o timeout_method=thread -x 2>&1 | tail -2
for cfg in A C; do
for mode in "BA_ATTN_1CTA=0 BA_ATTN_DEBUG=1" "BA_ATTN_1CTA=0" "BA_ATTN_1CTA=0 BA_EXP_EMU=1" "BA_ATTN_1CTA=0 BA_EXP_EMU=2"; do
  env $mode timeout 200 python bench.py --config $cfg --steps 5 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$cfg $mode','attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'clk',d['clocks']['sm_mhz'],d['clocks']['reasons'])" 2>&1 | tail -1
done; done
BA_ATTN_DEBUG=2 timeout 100 python bench.py --config A --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense 2>&1 | grep TRACE | head -9 > gpurun_out/trace2cta_v3.txt
