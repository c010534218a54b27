set -x
python -m pytest tests/test_gpu_parity.py -q -x -k "units or peers" 2>&1 | tail -5
python bench.py --config M --shard units --steps 3 --warmup 3 --no-cpu --no-e2e --no-dense 2>gpurun_out/units_M.err | tail -1 > gpurun_out/units_M.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --config M --shard units --fused --steps 3 --warmup 3 --no-cpu --no-e2e --no-dense 2>gpurun_out/units_M_fused.err | tail -1 > gpurun_out/units_M_fused.json
python - <<'PY'
import json
for f in ("units_M", "units_M_fused"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read())
        print(f, round(d["value"], 1), d["roofline"]["achieved"], d["gpu_launches"], d["config"]["parallelism"])
    except Exception as e:
        print(f, "ERR", e, open(f"gpurun_out/{f}.err").read()[-1500:])
PY
