sed -n 1,14p scripts/gpu_pptrace.sh > /tmp/h.sh; bash /tmp/h.sh
python -m pytest tests/test_gpu_parity.py -q -x -k "dissimilar or b128_kernel" 2>&1 | tail -1
for e in 2 1 3; do
  BA_PP_SEQ=1 BA_EXP_EMU=$e python bench.py --config A --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('SEQ emu=$e A', round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])"
done
python bench.py --config A --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('BASE A', round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])"
echo "== seq trace"; BA_PP_SEQ=1 BA_ATTN_DEBUG=2 python /tmp/tr.py A 1.0 2>&1 | grep TRACE
