for rep in 1 2 3; do
for lib in paper_2605_19726_b200/libbaatt.so build_ab/libbaatt_prev.so; do
  BA_LIB_PATH=$PWD/$lib timeout 200 python bench.py --config A --steps 20 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$lib sel',round(d['select_ms'],4))" 2>&1 | tail -1
done; done
