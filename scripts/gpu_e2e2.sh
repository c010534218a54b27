python -m pytest tests/test_gpu_parity.py -q -x -k "host_api" 2>&1 | tail -1
for c in A C V M; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'e2e/value', round(d['e2e']['value']/d['value'],3), d['clocks']['sm_mhz'])"
done
