mkdir -p gpurun_out/r1j
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_pp -c 1 -o gpurun_out/r1j/attn_A python bench.py --config A --profile --steps 1 --warmup 1 > /dev/null 2>&1; echo ncuA $?
timeout 600 ncu --set full --clock-control none -k regex:"gather_stats|scores|topk" -c 3 -o gpurun_out/r1j/select_M python bench.py --config M --profile --steps 1 --warmup 1 > /dev/null 2>&1; echo ncuM $?
ls -la gpurun_out/r1j
