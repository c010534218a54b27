timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 120 -o timeout_method=thread 2>&1 | tail -2
for cfg in C A; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gather_stats|norm_keys|radix|scores|topk" -c 40 --csv --log-file gpurun_out/launches_$cfg.csv python bench.py --config $cfg --profile --steps 1 --warmup 1 --no-e2e --no-dense --no-cpu > /dev/null 2>&1; echo ncu $cfg $?
timeout 200 python bench.py --config $cfg --steps 5 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/p2.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/p2.json'));print('$cfg','value',round(d['value'],1),'attn',round(d['roofline']['achieved'],1),'sel_ms',round(d['select_ms'],3),'share',round(d['select_share'],4))"
done
