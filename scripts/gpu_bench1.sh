set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; tail -3 gpurun_out/bench_c.err
cat gpurun_out/bench_c.json
timeout 200 python bench.py --config A --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; tail -3 gpurun_out/bench_a.err
cat gpurun_out/bench_a.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c.csv python bench.py --profile --steps 2 --warmup 1 --no-e2e --no-dense --no-cpu > /dev/null 2>&1; echo ncu1 $?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -c 1 -o gpurun_out/prof_attn_c python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_attn.log 2>&1; echo ncu2 $?; tail -3 gpurun_out/ncu_attn.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"norm_keys|radix|gather_stats|scores_kernel|topk" -c 14 -o gpurun_out/prof_sel_c python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_sel.log 2>&1; echo ncu3 $?; tail -3 gpurun_out/ncu_sel.log
