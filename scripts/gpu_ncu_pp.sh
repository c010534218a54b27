mkdir -p gpurun_out/pp
BA_ATTN_K5=pp timeout 400 ncu --set full --clock-control none --import-source on -k regex:attn_pp -c 1 -o gpurun_out/pp/pp_A python bench.py --config A --profile --steps 1 --warmup 1 > gpurun_out/pp/ncu.log 2>&1; echo ncu $?
tail -3 gpurun_out/pp/ncu.log
