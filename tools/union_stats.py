"""Union of the index lists of g adjacent (norm-sorted) query blocks, / kappa,
for g = 2 (the pair kernel's tile) and g = 4 (a 2-CTA cluster of pairs):
how much tensor work a shared K/V walk would waste on each workload."""
import sys, json, torch
sys.path.insert(0, '.')
from synth import CONFIGS, make_qkv
import paper_2605_19726_b200.baatt as ba
out = {}
for cfg in sys.argv[1:] or ["A", "C", "V", "M"]:
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda")
    ctx = ba.Context(q, k, v, w.block_size, w.density)
    sel = ctx.select(q, k, v)
    b, h, nq, kap = sel.kv_index.shape
    m = torch.zeros(b * h * nq, sel.n_k, dtype=torch.bool, device="cuda")
    m.scatter_(1, sel.kv_index.reshape(-1, kap).long(), True)
    m = m.reshape(b * h, nq, sel.n_k)
    r = {}
    for g in (2, 4, 8):
        n = nq // g
        u = m[:, :n * g].reshape(b * h, n, g, sel.n_k).any(2).sum(-1).double()
        r[f"union{g}_over_kappa"] = float(u.mean() / kap)
    out[cfg] = r
    del q, k, v, ctx, sel, m
    torch.cuda.empty_cache()
print(json.dumps(out))
