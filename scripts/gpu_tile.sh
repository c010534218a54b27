for t in 296 100; do
  BA_SCORES_TILE128_MIN=$t timeout 200 python bench.py --config A --steps 10 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('A tile128min=$t sel',round(d['select_ms'],3),'share',round(d['select_share'],4),'value',round(d['value'],1))" 2>&1 | tail -1
  BA_SCORES_TILE128_MIN=$t timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scores" -c 2 --csv python bench.py --config A --profile --steps 1 --warmup 0 --no-e2e --no-dense --no-cpu 2>/dev/null | grep scores | tail -1 | cut -d, -f5,15 | cut -c1-120
done
