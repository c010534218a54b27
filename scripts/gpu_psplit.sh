for lib in paper_2605_19726_b200/libbaatt.so build_ab/libbaatt_s4.so; do
for cfg in A C; do
  BA_LIB_PATH=$PWD/$lib timeout 200 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$lib $cfg',d['roofline']['kernel'],'attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
done; done
BA_LIB_PATH=$PWD/build_ab/libbaatt_s4.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "b128 or dissimilar" 2>&1 | tail -2
