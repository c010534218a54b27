mkdir -p gpurun_out/r1
# 1. launch list of the bench command (our kernels; cold-cache, serialised: compare shares)
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_sm100|gather_stats|norm_keys|radix|scores|topk" --csv --log-file gpurun_out/r1/launches_bench_C.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/r1/bench_profile_run.json 2>&1; echo ncu1 $?
# 2. full capture of the attention kernel at the bench workload
timeout 400 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -c 1 -o gpurun_out/r1/attn_C python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1; echo ncu2 $?
# 3. full capture of each selection kernel at the bench workload
timeout 500 ncu --set full --clock-control none -k regex:"gather_stats|norm_keys|radix_scatter|scores|topk" -c 9 -o gpurun_out/r1/select_C python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1; echo ncu3 $?
# 4. the bench itself (A and C), clocks recorded
timeout 300 python bench.py > gpurun_out/r1/bench_C.json 2> gpurun_out/r1/bench_C.err; cat gpurun_out/r1/bench_C.json
timeout 200 python bench.py --config A --no-cpu > gpurun_out/r1/bench_A.json 2>/dev/null; cat gpurun_out/r1/bench_A.json
timeout 200 python bench.py --config V --no-cpu > gpurun_out/r1/bench_V.json 2>/dev/null; cat gpurun_out/r1/bench_V.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r1/bench_ref.json 2>/dev/null; cat gpurun_out/r1/bench_ref.json
