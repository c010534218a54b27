# round-1 evidence refresh (pair kernel default, dual64, DMMA scores): launch list, full captures, bench lines
mkdir -p gpurun_out/r1e
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_pp|attn_sm100|gather_stats|norm_keys|radix|scores|topk" --csv --log-file gpurun_out/r1e/launches_bench_C.csv python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1; echo ncu1 $?
timeout 500 ncu --set full --clock-control none --import-source on -k regex:attn_pp -c 1 -o gpurun_out/r1e/attn_C python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1; echo ncu2 $?

timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_pp|attn_sm100|gather_stats|norm_keys|radix|scores|topk" --csv --log-file gpurun_out/r1e/launches_bench_M.csv python bench.py --config M --profile --steps 2 --warmup 1 > /dev/null 2>&1; echo ncu4 $?
timeout 400 python bench.py > gpurun_out/r1e/bench_C.json 2> gpurun_out/r1e/bench_C.err; cat gpurun_out/r1e/bench_C.json
for c in A V M; do timeout 300 python bench.py --config $c --no-cpu > gpurun_out/r1e/bench_$c.json 2>gpurun_out/r1e/bench_$c.err; cat gpurun_out/r1e/bench_$c.json; done
timeout 300 python bench.py --config C --density 0.25 --no-cpu --no-e2e > gpurun_out/r1e/bench_C25.json 2>/dev/null; cat gpurun_out/r1e/bench_C25.json
timeout 300 python bench.py --config C --top-p 0.9 --density 1.0 --no-cpu --no-e2e --no-dense > gpurun_out/r1e/bench_C_topp.json 2>/dev/null; cat gpurun_out/r1e/bench_C_topp.json
timeout 300 python bench.py --impl reference > gpurun_out/r1e/bench_ref.json 2>/dev/null; cat gpurun_out/r1e/bench_ref.json
timeout 400 python bench.py --config A --fidelity --no-cpu --no-e2e --no-dense > gpurun_out/r1e/bench_A_fidelity.json 2>/dev/null; cat gpurun_out/r1e/bench_A_fidelity.json
timeout 500 ncu --set full --clock-control none --import-source on -k regex:attn_sm100_kernel -c 1 -o gpurun_out/r1e/attn_M python bench.py --config M --profile --steps 1 --warmup 1 > /dev/null 2>&1; echo ncu5 $?
