python - <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_2605_19726_b200.baatt as ba
from synth import CONFIGS, make_qkv
w = CONFIGS["M"]
q, k, v = make_qkv(w, device="cuda")
ctx = ba.Context(q, k, v, 64, 0.5)
sel = ctx.select(q, k, v)
idx = sel.kv_index.long()
nk = sel.n_k
m = torch.zeros(idx.shape[0], idx.shape[1], idx.shape[2], nk, dtype=torch.bool, device="cuda")
m.scatter_(3, idx, True)
nq = m.shape[2] // 2 * 2
u = (m[:, :, 0:nq:2] | m[:, :, 1:nq:2]).sum(-1).float()
tiles = torch.ceil(u / 2)
useful = 2 * sel.kappa
print("M union/kappa", (u.mean() / sel.kappa).item(), "computed pairs per tile-CTA", (tiles * 4).mean().item(), "useful", useful, "useful fraction", (useful / (tiles * 4)).mean().item())
PY
