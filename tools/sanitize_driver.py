"""Small end-to-end calls for compute-sanitizer (memcheck / racecheck / synccheck):
ba_select on bf16 (K1 norm keys, K2 radix sort incl. windowed, K3 gather + stats,
K4 scores + top-kappa / top-p) and fp32 (config T), the SIMT attention (K6), and
the deviation / block-mass diagnostics' non-tcgen05 kernels.  Shapes are small
and ragged so every tail path runs.  Usage:
    compute-sanitizer --tool racecheck python tools/sanitize_driver.py [--tcgen05]
(--tcgen05 also runs the tensor-core attention kernels, which the sanitizer may
not model; off by default)."""
import sys
import torch
sys.path.insert(0, ".")
from synth import CONFIGS, make_qkv
import paper_2605_19726_b200.baatt as ba

tc = "--tcgen05" in sys.argv
for cfg, L, hq, hkv, B, kw in (("T", 1024 + 37, 1, 1, 64, {}),
                                ("A", 4096 + 77, 2, 1, 128, {}),
                                ("A", 4096 + 77, 2, 2, 128, {"sort_window": 1000}),
                                ("M", 2048 + 13, 2, 2, 64, {"top_p": 0.9})):
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    ctx = ba.Context(q, k, v, B, 0.5, sort_window=kw.get("sort_window", 0), top_p=kw.get("top_p"),
                     diagnostics=True)
    sel = ctx.select(q, k, v)
    if q.dtype == torch.float32 or tc:
        out = torch.empty_like(q)
        ctx.sparse_attn(out)
    if tc and q.dtype == torch.bfloat16 and ba.q_gather_supported(q, k, v, B):
        # NEXT-2 Q in place: the pair kernel's softmax warps load Q rows through pi_q
        zq = ba.Context(q, k, v, B, 0.5, zero_copy="q")
        zq.select(q, k, v)
        zq.sparse_attn(torch.empty_like(q))
    torch.cuda.synchronize()
    print(cfg, L, "ok", flush=True)
print("done")
