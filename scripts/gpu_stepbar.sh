#!/bin/bash
# per-step K/V full barrier: parity subset, skeleton, A/B vs per-item barriers
set -u
mkdir -p gpurun_out/sb
timeout 900 python -m pytest tests -m gpu -q -x -k "dissimilar or split_steps or b128 or smoke or pp or scatter or determinism or zero_copy or fullsize" > gpurun_out/sb/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/sb/pytest.txt
tail -3 gpurun_out/sb/pytest.txt
for d in 4 1; do
  BA_LIB_PATH=paper_2605_19726_b200/libbaatt_prof.so BA_ATTN_DEBUG=$d timeout 300 python bench.py --config A --steps 3 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/sb/skel_$d.json 2>/dev/null
  python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'attn', round(d['roofline']['achieved'],1), 'mhz', d['clocks']['sm_mhz'])" gpurun_out/sb/skel_$d.json "skeleton A mode=$d" 2>&1 | tail -1
done
bash scripts/gpu_ab.sh paper_2605_19726_b200/libbaatt_nosb.so "A C" none
bash scripts/gpu_ab.sh paper_2605_19726_b200/libbaatt_nosb.so "C" none "--random-lists --no-dense"
