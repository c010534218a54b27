#!/bin/bash
# selection A/B: product lib vs libbaatt_old.so — sel_ms at A / C / M (2 repeats), the selection parity subset,
# and the scores kernel's time and shared-memory bank conflicts at M (ncu)
set -u
mkdir -p gpurun_out/selab
timeout 900 python -m pytest tests -m gpu -q -x -k "selection or topk or fullsize or norm or perm or sort or window" > gpurun_out/selab/pytest.txt 2>&1; tail -1 gpurun_out/selab/pytest.txt
for r in 1 2; do for c in A C M; do for v in new old; do
  L=paper_2605_19726_b200/libbaatt.so; [ $v = old ] && L=paper_2605_19726_b200/libbaatt_old.so
  BA_LIB_PATH=$L timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/selab/${v}_$c.json 2>/dev/null
  python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'sel_ms', round(d['select_ms'],3), 'share', round(d['select_share'],4))" gpurun_out/selab/${v}_$c.json "$v $c"
done; done; done
for v in new old; do
  L=paper_2605_19726_b200/libbaatt.so; [ $v = old ] && L=paper_2605_19726_b200/libbaatt_old.so
  BA_LIB_PATH=$L timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:"topk_kernel" --csv python bench.py --config M --profile --no-e2e --no-cpu --no-dense --steps 1 --warmup 0 2>/dev/null | grep -E "duration" | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
done
