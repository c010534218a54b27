# launch lists of the current head for A and M (cold-cache, serialised)
mkdir -p gpurun_out/r1h
for cfg in A M V; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_|gather_stats|norm_keys|radix|scores|topk" --csv --log-file gpurun_out/r1h/launches_bench_$cfg.csv python bench.py --config $cfg --profile --steps 2 --warmup 1 > /dev/null 2>&1; echo ncu $cfg $?
python tools/launches.py gpurun_out/r1h/launches_bench_$cfg.csv > gpurun_out/r1h/launches_bench_$cfg.txt 2>&1; cat gpurun_out/r1h/launches_bench_$cfg.txt
done
