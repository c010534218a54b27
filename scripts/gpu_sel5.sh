timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "selection or topp or fp32" 2>&1 | tail -2
for cfg in A M C; do
  timeout 200 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$cfg','attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'sel',round(d['select_ms'],3),'share',round(d['select_share'],4),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gather_stats|norm_keys|radix|scores|topk" -c 40 --csv --log-file gpurun_out/sel_launches_A.csv python bench.py --config A --profile --steps 1 --warmup 1 --no-e2e --no-dense --no-cpu > /dev/null 2>&1; echo ncu $?
python tools/launches.py gpurun_out/sel_launches_A.csv 2>&1 | tail -11
