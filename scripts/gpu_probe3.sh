timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 120 -o timeout_method=thread -k "attention or dense or injected" 2>&1 | tail -2
for mode in "BA_ATTN_DEBUG=1" "BA_EXP_EMU=0" "BA_EXP_EMU=1" "BA_EXP_EMU=2"; do
  env $mode timeout 200 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/p2.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/p2.json'));print('$mode','attn_tflops',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'clk',d['clocks']['sm_mhz'])"
done
BA_ATTN_DEBUG=2 timeout 100 python bench.py --config A --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense 2>&1 | grep TRACE | head -15
