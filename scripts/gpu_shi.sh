timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "pp or bf16 or zero_copy or topp or dissimilar" 2>&1 | tail -2 > gpurun_out/shi_tests.txt
for cfg in A C V; do
  timeout 200 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$cfg',d['roofline']['kernel'],'attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
done
cat gpurun_out/shi_tests.txt
