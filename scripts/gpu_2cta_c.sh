for mode in "BA_ATTN_1CTA=1 BA_ATTN_DEBUG=1" "BA_ATTN_1CTA=0 BA_ATTN_DEBUG=1" "BA_ATTN_1CTA=1" "BA_ATTN_1CTA=0" "BA_ATTN_1CTA=0 BA_EXP_EMU=1" "BA_ATTN_1CTA=0 BA_EXP_EMU=2" "BA_ATTN_1CTA=1 BA_EXP_EMU=1"; do
  env $mode timeout 200 python bench.py --config A --steps 5 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('A $mode','attn',round(d['roofline']['achieved'],1),'clk',d['clocks']['sm_mhz'],d['clocks']['reasons'])"
done
