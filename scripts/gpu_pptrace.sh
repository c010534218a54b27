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
for e in 1 0; do
echo "== A emu=$e"; BA_EXP_EMU=$e BA_ATTN_DEBUG=2 python /tmp/tr.py A 2>&1 | grep TRACE
done
echo "== A dense"; BA_ATTN_DEBUG=2 python /tmp/tr.py A 1.0 2>&1 | grep TRACE
