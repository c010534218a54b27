"""Diagnostic: inject random (dissimilar) kv lists and report per-block errors."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_19726_b200.baatt as ba
from synth import CONFIGS, make_qkv
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from parity import oracle_output_with_gpu_selection

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
w = CONFIGS["A" if B == 128 else "M"]
L = 16 * B
q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=2, heads_kv=2)
ctx = ba.Context(q, k, v, B, 0.5)
sel = ctx.select(q, k, v)
rng = np.random.default_rng(3)
idx = np.sort(np.stack([np.stack([rng.choice(16, 8, replace=False) for _ in range(16)]) for _ in range(2)]), axis=-1)
sel.kv_index.copy_(torch.from_numpy(idx[None].astype(np.int32)))
out = torch.empty_like(q)
ctx.sparse_attn(out)
torch.cuda.synchronize()
ref = oracle_output_with_gpu_selection(q, k, v, sel, B)
pq = sel.perm_q.cpu().numpy()
g = out.double().cpu().numpy()
print("kernel", ba.attention_kernel_name(q, k, v, B))
for h in range(2):
    errs = []
    for blk in range(16):
        s, e = blk * B, (blk + 1) * B
        rows = pq[0, h, s:e]
        errs.append(np.abs(g[0, h, rows] - ref[0, h, rows]).max())
    print("head", h, " ".join(f"{x:.3f}" for x in errs))
    if h == 0:
        for p in range(3):
            a_, b_ = set(idx[h, 2 * p]), set(idx[h, 2 * p + 1])
            print("  pair", p, "A", sorted(a_), "B", sorted(b_))
