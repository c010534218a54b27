# B = 64 dual tiles: parity + M bench dual vs pair; pp (reverted single-pass) vs 1cta at A
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "B64 or dissimilar or topp or full_density" 2>&1 | tail -4
for mode in "BA_ATTN_B64=dual" "BA_ATTN_B64=pair" "BA_ATTN_B64=dual BA_ATTN_DEBUG=1"; do
  env $mode timeout 200 python bench.py --config M --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('M $mode','attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'sel',round(d['select_ms'],3),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
  tail -1 gpurun_out/p.err
done
for mode in "BA_ATTN_K5=pp" "BA_ATTN_K5=1cta"; do
  env $mode timeout 200 python bench.py --config A --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('A $mode','attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
done
