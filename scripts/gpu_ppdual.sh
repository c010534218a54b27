timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "pp_dual64 or ppdual" 2>&1 | tail -3 > gpurun_out/ppd_tests.txt
for mode in "BA_ATTN_B64=ppdual" "BA_ATTN_B64=dual"; do
  env $mode timeout 200 python bench.py --config M --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('M $mode',d['roofline']['kernel'],'attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
  tail -1 gpurun_out/p.err
done
cat gpurun_out/ppd_tests.txt
