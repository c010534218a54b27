#!/bin/bash
# Selection kernels at config A: launch list + one full ncu capture of each selection kernel.
set -u
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/sel_launches_A.csv python bench.py --config A --profile --no-e2e --no-cpu --no-dense --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/sel_launches_A.csv 2>&1 | grep baatt
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:keys_hist|onesweep|gather_stats|scores_topk" -c 7 -o gpurun_out/sel_A_full python bench.py --config A --profile --no-e2e --no-cpu --no-dense --steps 1 --warmup 0 > gpurun_out/sel_full.log 2>&1
ls -la gpurun_out/sel_A_full.ncu-rep
