timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "host or attention" 2>&1 | tail -2
for cfg in C A; do
timeout 300 python bench.py --config $cfg --no-cpu --no-dense > gpurun_out/e2e.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/e2e.json'));print('$cfg value',round(d['value'],1),'e2e',d['e2e'])"
done
