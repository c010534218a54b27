python -m pytest tests/test_gpu_parity.py -q -x -k "dissimilar or b128_kernel or units or peers or zero_copy or attention_bf16 or dense" 2>&1 | tail -2
python - <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_2605_19726_b200.baatt as ba
from synth import CONFIGS, make_qkv
for cfg in ("A", "C", "V"):
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", heads_q=8, heads_kv=min(8, w.heads_kv))
    ctx = ba.Context(q, k, v, w.block_size, 0.5)
    sel = ctx.select(q, k, v)
    idx = sel.kv_index.long()
    m = torch.zeros(idx.shape[0], idx.shape[1], idx.shape[2], sel.n_k, dtype=torch.bool, device="cuda")
    m.scatter_(3, idx, True)
    nq = m.shape[2] // 2 * 2
    u = (m[:, :, 0:nq:2] | m[:, :, 1:nq:2]).sum(-1).float()
    print(cfg, "pair union / kappa", round((u.mean() / sel.kappa).item(), 4))
    del q, k, v, ctx, sel, m
PY
for i in 1 2; do for c in A C; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c', round(d['roofline']['achieved'],1), round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
BA_PP_SEQ=1 BA_EXP_EMU=2 python bench.py --config A --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('SEQ A', round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])"
