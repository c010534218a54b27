python -m pytest tests/test_gpu_parity.py -q -x -k "b128_kernel and pp" 2>&1 | tail -1
for i in 1 2; do
for c in A C; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c', round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
