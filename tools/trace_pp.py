"""Tile timeline of the pair kernel (profiling build only).

    python -m paper_2605_19726_b200.build --profiling --out paper_2605_19726_b200/libbaatt_prof.so
    BA_LIB_PATH=paper_2605_19726_b200/libbaatt_prof.so BA_ATTN_DEBUG=2 python tools/trace_pp.py [A|C] [--dense]

CTA (0, 0) prints clock64 stamps of steps kTraceStart .. +8 (attn_sm100_pp.cu, kMode 2)
of one full-size launch; this script prints per-step deltas between the stamps.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(cfg: str, dense: bool):
    import torch
    import paper_2605_19726_b200.baatt as ba
    from synth import CONFIGS, make_qkv
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda")
    ctx = ba.Context(q, k, v, w.block_size, 1.0 if dense else w.density)
    ctx.select(q, k, v)
    out = torch.empty_like(q)
    torch.cuda.synchronize()
    ctx.sparse_attn(out)
    torch.cuda.synchronize()


def main():
    if os.environ.get("BA_TRACE_CHILD"):
        run(sys.argv[1], "--dense" in sys.argv)
        return
    env = dict(os.environ, BA_TRACE_CHILD="1")
    r = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True, text=True)
    rows = {}
    for line in r.stdout.splitlines():
        if line.startswith("TRACE"):
            parts = line.split()
            rows[parts[1]] = [int(x) for x in parts[2:]]
    if not rows:
        print(r.stdout[-2000:], r.stderr[-2000:])
        sys.exit(1)
    names = list(rows)
    n = min(len(v) for v in rows.values())
    print("raw stamps (cycles from CTA start):")
    for k in names:
        print(f"  {k:9s}", " ".join(f"{x:8d}" for x in rows[k][:n]))
    print("per-step period (A_wait[j+1] - A_wait[j]):", [rows["A_wait"][j + 1] - rows["A_wait"][j] for j in range(n - 1)])
    for x in "AB":
        W, L, P0, E = (rows[x + t] for t in ("_wait", "_ld", "_p0", "_end"))
        print(f"softmax {x}: S ready -> ld done {[L[j] - W[j] for j in range(n)]}")
        print(f"           ld -> P part 0 published {[P0[j] - L[j] for j in range(n)]}")
        print(f"           part 0 -> end (part 1 + sums) {[E[j] - P0[j] for j in range(n)]}")
        print(f"           end -> next S ready {[W[j + 1] - E[j] for j in range(n - 1)]}")

if __name__ == "__main__":
    main()
