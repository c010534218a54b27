"""Full-size parity at the BASELINE.json configurations, in the launch
configuration bench.py times (Context.select + Context.sparse_attn on the full
tensors).

The oracle cannot run every head of a 128K problem in seconds, so:
  * selection (P1, P4) is checked in full for sampled q-heads (first and last,
    i.e. different GQA groups), every query block of those heads;
  * outputs (P5) are checked on sampled query blocks of those heads — block 0,
    the last (ragged for config V) block, the block with the most
    near-threshold entries and a seeded random one — computed by the oracle
    one block at a time with the GPU's permutations and index lists;
  * properties that hold at any size are checked on the whole output:
    kv_count == kappa, index rows strictly ascending and in range, finite
    output, permutations are bijections.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
from synth import CONFIGS, make_qkv

from parity import MASK_BAND, TOL, check_selection, oracle_select_all

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def ba():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_19726_b200.baatt as ba
    ba.load()
    return ba


def _blocks_to_check(ref, nq, seed):
    near = (np.abs(ref.m - ref.tau[:, None]) <= 1e-4).sum(axis=1)
    rng = np.random.default_rng(seed)
    return sorted({0, nq - 1, int(near.argmax()), int(rng.integers(nq))})


@pytest.mark.parametrize("cfg,density,top_p", [("A", 0.5, None), ("C", 0.5, None), ("C", 0.25, None), ("V", 0.5, None),
                                              ("M", 0.5, None), ("C", 1.0, 0.9), ("M", 0.5, 0.95)])
def test_fullsize(ba, cfg, density, top_p):
    w = CONFIGS[cfg]
    torch.cuda.empty_cache()
    q, k, v = make_qkv(w, device="cuda")
    if top_p is not None:
        top_p = float(np.float32(top_p))  # the ABI carries top_p as fp32
    ctx = ba.Context(q, k, v, w.block_size, density, 1.0, "qk", "diag", top_p=top_p)
    out = torch.empty_like(q)
    sel = ctx.select(q, k, v)
    ctx.sparse_attn(out)
    torch.cuda.synchronize()
    kappa, nq, nk = sel.kappa, sel.n_q, sel.n_k
    # ---- properties over the whole problem
    cnt = sel.kv_count.long()
    if top_p is None:
        assert (cnt == kappa).all()
    else:
        assert (cnt >= 1).all() and (cnt <= kappa).all()
    idx = sel.kv_index.long()
    valid = torch.arange(kappa, device="cuda") < cnt[..., None]
    assert ((idx >= 0) & (idx < nk) | ~valid).all()
    assert ((idx[..., 1:] > idx[..., :-1]) | ~valid[..., 1:]).all()
    assert torch.isfinite(out.float()).all()
    for perm in (sel.perm_q, sel.perm_k):
        srt = torch.sort(perm.long(), dim=-1).values
        assert torch.equal(srt, torch.arange(perm.shape[-1], device="cuda").expand_as(srt))
    # ---- selection of sampled heads vs the oracle (every query block)
    heads = sorted({0, w.heads_q - 1})
    ref = oracle_select_all(q, k, w.block_size, density, 1.0, "qk", "diag", heads=heads, top_p=top_p)
    rep = check_selection(sel, ref)
    # ---- sampled output blocks vs the oracle (GPU perm + index lists)
    grp = w.heads_q // w.heads_kv
    scale = 1.0 / math.sqrt(w.head_dim)
    worst = 0.0
    for h in heads:
        hk = h // grp
        pq = sel.perm_q[0, h].cpu().numpy()
        pk = sel.perm_k[0, hk].cpu().numpy()
        kvi_all = sel.kv_index[0, h].cpu().numpy()
        kvc = sel.kv_count[0, h].cpu().numpy()
        kvi = [kvi_all[g, :kvc[g]] for g in range(nq)]
        Qs = O.apply_permutation(q[0, h].cpu(), pq)
        Ks = O.apply_permutation(k[0, hk].cpu(), pk)
        Vs = O.apply_permutation(v[0, hk].cpu(), pk)
        blocks = _blocks_to_check(ref[(0, h)], nq, seed=h)
        Os, _ = O.block_sparse_attention_head(Qs, Ks, Vs, kvi, w.block_size, scale, blocks)
        gout = out[0, h].float().cpu().numpy()
        for g in blocks:
            s, e = g * w.block_size, min((g + 1) * w.block_size, q.shape[2])
            rows = pq[s:e]  # original positions of the sorted rows of this block
            err = np.abs(gout[rows] - Os[s:e]).max()
            worst = max(worst, float(err))
    assert worst <= TOL[q.dtype], (worst, rep)


def test_max_length_one_million_tokens(ba):
    """Maximum size of the pair kernel's bitmask (N_k = 8192 key blocks: L = 2^20
    tokens, B = 128), 5% density: selection of the head vs the oracle (every
    query block, within the band), sampled output blocks vs the oracle, and the
    whole-problem properties."""
    w = CONFIGS["A"]
    L = 1 << 20
    torch.cuda.empty_cache()
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=1, heads_kv=1)
    assert ba.attention_kernel_name(q, k, v, 128) == "attn_sm100_tcgen05_pp"
    ctx = ba.Context(q, k, v, 128, 0.05)
    sel = ctx.select(q, k, v)
    out = torch.empty_like(q)
    ctx.sparse_attn(out)
    torch.cuda.synchronize()
    assert sel.n_k == 8192 and (sel.kv_count == sel.kappa).all()
    assert torch.isfinite(out.float()).all()
    ref = oracle_select_all(q, k, 128, 0.05, 1.0, "qk", "diag")
    check_selection(sel, ref)
    pq, pk = sel.perm_q[0, 0].cpu().numpy(), sel.perm_k[0, 0].cpu().numpy()
    kvi = sel.kv_index[0, 0].cpu().numpy()
    Qs, Ks, Vs = (O.apply_permutation(t[0, 0].cpu(), p) for t, p in ((q, pq), (k, pk), (v, pk)))
    blocks = _blocks_to_check(ref[(0, 0)], sel.n_q, seed=7)
    Os, _ = O.block_sparse_attention_head(Qs, Ks, Vs, kvi, 128, 1.0 / math.sqrt(128), blocks)
    gout = out[0, 0].float().cpu().numpy()
    for g in blocks:
        rows = pq[g * 128:(g + 1) * 128]
        assert np.abs(gout[rows] - Os[g * 128:(g + 1) * 128]).max() <= TOL[q.dtype]


@pytest.mark.parametrize("cfg,world", [("M", 8), ("C", 3)])
def test_unit_split_full_size_bitwise(ba, cfg, world):
    """SURVEY 8(e) at full size: config M's 28 heads on 8 simulated ranks (and C's
    8 GQA groups on 3, splitting a group) — each rank selects over the heads its
    (head, q-block) units touch and runs ba_sparse_attn_units; the union of the
    ranks' rows equals the 1-GPU output bit for bit."""
    from paper_2605_19726_b200.dist import unit_heads, unit_range
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda")
    ref = torch.empty_like(q)
    ctx = ba.Context(q, k, v, w.block_size, w.density)
    ctx.select(q, k, v)
    ctx.sparse_attn(ref)
    nq = ctx.sel.n_q
    del ctx
    out = torch.full_like(q, float("nan"))
    sizes = []
    for r in range(world):
        u0, u1 = unit_range(w.heads_q, nq, world, r)
        sizes.append(u1 - u0)
        q0, q1, k0, k1 = unit_heads(u0, u1, nq, w.heads_q, w.heads_kv)
        qs, ks, vs = q[:, q0:q1].contiguous(), k[:, k0:k1].contiguous(), v[:, k0:k1].contiguous()
        c = ba.Context(qs, ks, vs, w.block_size, w.density, out=out[:, q0:q1])
        c.select(qs, ks, vs)
        c.sparse_attn_units(u0 - q0 * nq, u1 - q0 * nq, [out[:, q0:q1]])
        del c, qs, ks, vs
    torch.cuda.synchronize()
    assert max(sizes) - min(sizes) <= 2
    assert torch.equal(out, ref)
