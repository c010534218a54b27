#!/bin/bash
# Pair-kernel skeleton ceilings (profiling build): BA_ATTN_DEBUG 0 product, 1 no softmax, 3 no softmax + no loads,
# 4 also no P stores, 5 full softmax + no loads.  Attention TF/s from bench (numbers of modes 1-5 are timing only).
set -u
mkdir -p gpurun_out/skel
for c in C A; do
  for dn in 0.5 1.0; do
    for d in 0 1 3 4 5; do
      BA_LIB_PATH=paper_2605_19726_b200/libbaatt_prof.so BA_ATTN_DEBUG=$d timeout 300 python bench.py --config $c --density $dn --steps 3 --warmup 2 --no-e2e --no-cpu --no-dense > gpurun_out/skel/${c}_${dn}_$d.json 2> gpurun_out/skel/${c}_${dn}_$d.err
      python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], 'attn', round(d['roofline']['achieved'],1), 'mhz', d['clocks']['sm_mhz'])" gpurun_out/skel/${c}_${dn}_$d.json "$c rho=$dn mode=$d" 2>&1 | tail -1
    done
  done
done
