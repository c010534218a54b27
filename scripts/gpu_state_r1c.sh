# re-entry state check: full gpu suite, then A/C bench for default vs pp kernel
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -x 2>&1 | tail -3
for cfg in A C M; do
for mode in "BA_ATTN_K5=1cta" "BA_ATTN_K5=pp" "BA_ATTN_K5=pp BA_ATTN_DEBUG=1" "BA_ATTN_DEBUG=1"; do
  env $mode timeout 200 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$cfg $mode','attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'sel_ms',round(d['select_ms'],3),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
  tail -1 gpurun_out/p.err
done; done
