python -m pytest tests/test_gpu_parity.py -q -x -k "dissimilar or b128_kernel" 2>&1 | tail -1
for i in 1 2; do for c in A C; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c', round(d['roofline']['achieved'],1), round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
