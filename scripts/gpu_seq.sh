cat > /tmp/tr.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_2605_19726_b200.baatt as ba
from synth import CONFIGS, make_qkv
w = CONFIGS[sys.argv[1]]
q, k, v = make_qkv(w, device="cuda", heads_q=4, heads_kv=min(4, w.heads_kv))
dens = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
ctx = ba.Context(q, k, v, w.block_size, dens)
ctx.select(q, k, v)
out = torch.empty_like(q)
ctx.sparse_attn(out)
torch.cuda.synchronize()
PY
python -m pytest tests/test_gpu_parity.py -q -x -k "dissimilar or b128_kernel" 2>&1 | tail -3
for e in 1 0 2 3; do
  BA_PP_SEQ=1 BA_EXP_EMU=$e python bench.py --config A --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('SEQ emu=$e A', round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])"
done
python bench.py --config A --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('BASE A', round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])"
echo "== seq trace"; BA_PP_SEQ=1 BA_ATTN_DEBUG=2 python /tmp/tr.py A 1.0 2>&1 | grep TRACE
