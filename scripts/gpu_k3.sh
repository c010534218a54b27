python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "selection or B64 or M or stats or units" 2>&1 | tail -2
for i in 1 2; do
python bench.py --config M --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('M sel', round(d['select_ms'],3), 'value', round(d['value'],1), d['clocks']['sm_mhz'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gather_stats" --csv --log-file gpurun_out/k3_M.csv python bench.py --config M --profile --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/k3_M.csv
