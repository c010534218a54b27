set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "selection or fullsize or topp or windowed or fused or deterministic" > gpurun_out/pytest_sel.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_sel.txt
tail -3 gpurun_out/pytest_sel.txt; grep MULTICAST -r gpurun_out/ 2>/dev/null | head -2
for c in A C; do
  timeout 300 python bench.py --config $c --no-e2e --no-cpu --no-dense --steps 5 --warmup 3 > gpurun_out/sel_$c.json 2> gpurun_out/sel_$c.err
  python -c "import json; d=json.load(open('gpurun_out/sel_$c.json')); print('$c', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'sel_ms', round(d['select_ms'],3), 'share', round(d['select_share'],4), 'launches/step', d['gpu_launches']/d['steps'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/sel_launches_A.csv python bench.py --config A --profile --no-e2e --no-cpu --no-dense --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/sel_launches_A.csv 2>/dev/null | grep baatt
