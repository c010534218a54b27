# parity (bf16 + fp32), then exp2-offload sweep at config C, then selection-kernel profile
timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 120 -o timeout_method=thread 2>&1 | tail -4
for e in 0 1 2 3 4; do
  BA_EXP_EMU=$e timeout 200 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/emu_$e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/emu_$e.json'));print('emu',$e,'value',round(d['value'],1),'attn_tflops',round(d['roofline']['achieved'],1),'frac',round(d['roofline']['frac'],3),'sel_ms',round(d['select_ms'],2),'clk',d['clocks'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:baatt -c 60 --csv --log-file gpurun_out/launches_c.csv python bench.py --profile --steps 2 --warmup 1 --no-e2e --no-dense --no-cpu > /dev/null 2>&1; echo ncu $?
