for i in 1 2; do
for lib in tools/libbaatt_old.so paper_2605_19726_b200/libbaatt.so; do
  BA_LIB_PATH=$PWD/$lib timeout 200 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$lib','attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'clk',d['clocks']['sm_mhz'])"
done; done
