mkdir -p gpurun_out/r1b
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_sm100|gather_stats|norm_keys|radix|scores|topk" --csv --log-file gpurun_out/r1b/launches_bench_C.csv python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1; echo ncu1 $?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -c 1 -o gpurun_out/r1b/attn_C python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1; echo ncu2 $?
timeout 500 ncu --set full --clock-control none -k regex:"scores_kernel|topk_kernel" -c 2 -o gpurun_out/r1b/select2_C python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1; echo ncu3 $?
timeout 300 python bench.py > gpurun_out/r1b/bench_C.json 2> gpurun_out/r1b/bench_C.err; cat gpurun_out/r1b/bench_C.json
for c in A V M; do timeout 300 python bench.py --config $c --no-cpu > gpurun_out/r1b/bench_$c.json 2>/dev/null; done
timeout 300 python bench.py --impl reference > gpurun_out/r1b/bench_ref.json 2>/dev/null; cat gpurun_out/r1b/bench_ref.json
