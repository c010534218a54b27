#!/bin/bash
# dual-issue pair kernel: parity subset, skeleton ceilings, A/B vs single issuer
set -u
mkdir -p gpurun_out/dual
timeout 900 python -m pytest tests -m gpu -q -x -k "dissimilar or split_steps or b128 or smoke or pp or scatter or determinism" > gpurun_out/dual/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/dual/pytest.txt
tail -3 gpurun_out/dual/pytest.txt
for d in 4 1 5; do
  BA_LIB_PATH=paper_2605_19726_b200/libbaatt_prof.so BA_ATTN_DEBUG=$d timeout 300 python bench.py --config A --steps 3 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/dual/skel_$d.json 2>/dev/null
  python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'attn', round(d['roofline']['achieved'],1), 'mhz', d['clocks']['sm_mhz'])" gpurun_out/dual/skel_$d.json "skeleton A mode=$d" 2>&1 | tail -1
done
bash scripts/gpu_ab.sh paper_2605_19726_b200/libbaatt_single.so "A C" none
