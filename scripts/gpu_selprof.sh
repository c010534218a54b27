# selection kernels at A: launch list + pipe utilisation
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gather_stats|norm_keys|radix|scores|topk" -c 40 --csv --log-file gpurun_out/sel_launches_A.csv python bench.py --config A --profile --steps 1 --warmup 1 --no-e2e --no-dense --no-cpu > /dev/null 2>&1; echo ncu $?
python tools/launches.py gpurun_out/sel_launches_A.csv 2>&1 | tail -14
timeout 300 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio --clock-control none -k regex:"gather_stats|norm_keys" -c 5 --csv --log-file gpurun_out/sel_pipes_A.csv python bench.py --config A --profile --steps 1 --warmup 0 --no-e2e --no-dense --no-cpu > /dev/null 2>&1; echo ncu2 $?
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/sel_pipes_A.csv'))]
hdr=None
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); print(d['ID'], d['Kernel Name'][:40], d['Metric Name'][:60], d['Metric Value'])
PY
