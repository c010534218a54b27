#!/bin/bash
# Pair-kernel tile timelines (profiling builds): reload vs no-reload, sparse and dense, configs A and C.
set -u
mkdir -p gpurun_out/trace
for lib in prof prof0; do
  for c in A C; do
    for m in "" "--dense"; do
      BA_LIB_PATH=paper_2605_19726_b200/libbaatt_$lib.so BA_ATTN_DEBUG=2 timeout 300 python tools/trace_pp.py $c $m > gpurun_out/trace/${lib}_${c}${m}.txt 2>&1
      echo "== $lib $c $m"; tail -9 gpurun_out/trace/${lib}_${c}${m}.txt
    done
  done
done
