# top-p parity; pp kernel tile trace and exp-offload sweep at A (no power cap there)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "topp" 2>&1 | tail -15
BA_ATTN_K5=pp BA_ATTN_DEBUG=2 timeout 200 python bench.py --config A --steps 1 --warmup 0 --no-e2e --no-cpu --no-dense 2>&1 | grep TRACE | head -14
BA_ATTN_DEBUG=2 timeout 200 python bench.py --config A --steps 1 --warmup 0 --no-e2e --no-cpu --no-dense 2>&1 | grep TRACE | head -16
for mode in "BA_ATTN_K5=pp BA_EXP_EMU=1" "BA_ATTN_K5=pp BA_EXP_EMU=2" "BA_ATTN_K5=pp BA_EXP_EMU=3" "BA_ATTN_K5=pp"; do
  env $mode timeout 200 python bench.py --config A --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('A $mode','attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
done
