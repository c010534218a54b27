for sk in 0 1 2 3; do
  BA_ATTN_DEBUG=1 BA_ATTN_SKIPLOAD=$sk timeout 200 python bench.py --config A --steps 5 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('no-softmax skipload=$sk','attn',round(d['roofline']['achieved'],1),'clk',d['clocks']['sm_mhz'])"
done
