python -m pytest tests/test_gpu_parity.py -q -x -k "selection" 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scores" --csv --log-file gpurun_out/sc_M.csv python bench.py --config M --profile --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/sc_M.csv
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scores" --csv --log-file gpurun_out/sc_C.csv python bench.py --config C --profile --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/sc_C.csv
