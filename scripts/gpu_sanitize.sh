#!/bin/bash
# (compute-sanitizer has since been closed on the GPU pool: the runs kept in profiles/ are from round 2, e541b0c)
# compute-sanitizer memcheck / racecheck / synccheck on the selection kernels (K1-K4) and the
# SIMT attention (K6) over small ragged problems (tools/sanitize_driver.py); summaries -> gpurun_out/
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --target-processes all --print-limit 50 python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.txt
done
timeout 1200 $CS --tool memcheck --target-processes all --print-limit 50 python tools/sanitize_driver.py --tcgen05 > gpurun_out/sanitize_memcheck_tcgen05.txt 2>&1
echo "rc=$?" >> gpurun_out/sanitize_memcheck_tcgen05.txt
for f in gpurun_out/sanitize_*.txt; do echo "== $f"; tail -3 "$f"; done
