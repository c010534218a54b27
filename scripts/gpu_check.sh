#!/bin/bash
# One GPU call: the GPU test suite, smoke(), and a short default bench line.
#   gpurun --timeout 2400 -- bash scripts/gpu_check.sh [pytest -k expr]
set -u
mkdir -p gpurun_out
K=${1:-}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [ -n "$K" ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
else
  timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C.json 2> gpurun_out/bench_C.err
tail -3 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/smoke.txt; head -c 600 gpurun_out/bench_C.json
