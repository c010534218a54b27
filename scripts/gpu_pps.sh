timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "pps" 2>&1 | tail -8
for cfg in A C; do
for mode in "BA_ATTN_K5=pps" "BA_ATTN_K5=pps BA_EXP_EMU=0" "BA_ATTN_K5=pps BA_EXP_EMU=2" "BA_ATTN_K5=pp"; do
  env $mode timeout 200 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$cfg $mode',d['roofline']['kernel'],'attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
  tail -1 gpurun_out/p.err
done; done
