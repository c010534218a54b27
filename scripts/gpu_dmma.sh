nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dm tools/dmma_bench.cu && /tmp/dm
for cfg in M C; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gather_stats|norm_keys|radix|scores|topk" -c 40 --csv --log-file gpurun_out/sel_launches_$cfg.csv python bench.py --config $cfg --profile --steps 1 --warmup 1 --no-e2e --no-dense --no-cpu > /dev/null 2>&1; echo ncu $cfg $?
python tools/launches.py gpurun_out/sel_launches_$cfg.csv 2>&1 | tail -11
done
