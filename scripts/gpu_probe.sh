./tools/microbench
BA_ATTN_DEBUG=1 timeout 200 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/dbg1.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/dbg1.json'));print('NO-SOFTMAX attn_tflops',round(d['roofline']['achieved'],1),'clk',d['clocks'])"
BA_ATTN_DEBUG=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -c 1 -o gpurun_out/prof_attn_nosoftmax python bench.py --profile --steps 1 --warmup 1 --config A > /dev/null 2>&1; echo ncu $?
BA_EXP_EMU=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -c 1 -o gpurun_out/prof_attn_v2 python bench.py --profile --steps 1 --warmup 1 --config A > /dev/null 2>&1; echo ncu $?
