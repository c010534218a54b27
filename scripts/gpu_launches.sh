for cfg in C A; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_sm100|gather_stats|norm_keys|radix|scores|topk" -c 40 --csv --log-file gpurun_out/launches_$cfg.csv python bench.py --config $cfg --profile --steps 1 --warmup 1 --no-e2e --no-dense --no-cpu > /dev/null 2>&1; echo ncu $cfg $?
done
