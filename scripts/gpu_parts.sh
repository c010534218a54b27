timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "B64 or dissimilar or b128 or zero_copy or peers or fp32 or bf16" 2>&1 | tail -2 > gpurun_out/parts_tests.txt
for mode in "BA_ATTN_B64=dual" "BA_ATTN_B64=pair"; do
  env $mode timeout 200 python bench.py --config M --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('M $mode',d['roofline']['kernel'],'attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'clk',(d['clocks'] or {}).get('sm_mhz'))" 2>&1 | tail -1
done
BA_ATTN_K5=1cta timeout 200 python bench.py --config A --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
python -c "import json;d=json.load(open('gpurun_out/p.json'));print('A 1cta',d['roofline']['kernel'],'attn',round(d['roofline']['achieved'],1))"
cat gpurun_out/parts_tests.txt
