timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "selection or topp or fp32 or exact or zero_copy" 2>&1 | tail -1 > gpurun_out/gm_tests.txt
for cfg in A M; do
  timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$cfg sel',round(d['select_ms'],3),'share',round(d['select_share'],4),'value',round(d['value'],1))" 2>&1 | tail -1
done
cat gpurun_out/gm_tests.txt
