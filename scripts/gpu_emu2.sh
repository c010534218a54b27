for e in 0 1 2 3; do
for cfg in A C; do
  BA_EXP_EMU=$e timeout 200 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$cfg EMU=$e attn',round(d['roofline']['achieved'],1),'value',round(d['value'],1),'clk',(d['clocks'] or {}).get('sm_mhz'),(d['clocks'] or {}).get('reasons'))" 2>&1 | tail -1
done; done
python - <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_2605_19726_b200.baatt as ba
from synth import CONFIGS, make_qkv
for cfg in ("A", "C"):
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda")
    ctx = ba.Context(q, k, v, w.block_size, w.density)
    sel = ctx.select(q, k, v)
    idx = sel.kv_index.long()  # [b, h, nq, kappa]
    nk = sel.n_k
    m = torch.zeros(idx.shape[0], idx.shape[1], idx.shape[2], nk, dtype=torch.bool, device="cuda")
    m.scatter_(3, idx, True)
    nq = m.shape[2] // 2 * 2
    u = (m[:, :, 0:nq:2] | m[:, :, 1:nq:2]).sum(-1).float()
    print(cfg, "union/kappa", (u.mean() / sel.kappa).item(), "useful fraction", (2 * sel.kappa / (2 * u)).mean().item())
PY
