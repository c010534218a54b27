"""GPU parity tests: CUDA path through the C ABI vs the fp64 oracle.

Run on a B200 with `pytest -m gpu`.  Inputs are seeded synthetic tensors
(synth/, recipe in DESIGN.md); the oracle always receives the exact tensors the
GPU consumed.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
from synth import CONFIGS, make_qkv

from parity import (TOL, check_selection, max_abs_err, oracle_output_with_gpu_selection,
                    oracle_select_all)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ba():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_19726_b200.baatt as ba
    ba.load()
    return ba


def _run_select(ba, q, k, v, B, density, beta=1.0, sort="qk", comp="diag", window=0):
    ctx = ba.Context(q, k, v, B, density, beta, sort, comp, window, diagnostics=True)
    sel = ctx.select(q, k, v)
    torch.cuda.synchronize()
    return ctx, sel


# ---------------------------------------------------------------- selection (P1-P4)
@pytest.mark.parametrize("sort", ["qk", "none", "q", "k"])
def test_selection_tiny_T(ba, sort):
    w = CONFIGS["T"]
    q, k, v = make_qkv(w, device="cuda")
    _, sel = _run_select(ba, q, k, v, w.block_size, w.density, sort=sort)
    ref = oracle_select_all(q, k, w.block_size, w.density, 1.0, sort, "diag")
    rep = check_selection(sel, ref)
    assert rep["max_stat_err"] < 1e-12
    # keys bit-exact (reading A4)
    np.testing.assert_array_equal(sel.q_key.cpu().numpy()[0, 0], O.norm_key(q[0, 0].cpu()))


@pytest.mark.parametrize("cfg,L,hq,hkv,dens,comp", [
    ("A", 4096 + 77, 4, 4, 0.5, "diag"),
    ("C", 8192, 8, 2, 0.25, "diag"),
    ("C", 3000, 4, 1, 0.5, "none"),
    ("M", 4096 + 13, 3, 3, 0.5, "diag"),
    ("V", 4500, 2, 2, 0.4, "diag"),
])
def test_selection_bf16(ba, cfg, L, hq, hkv, dens, comp):
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    _, sel = _run_select(ba, q, k, v, w.block_size, dens, comp=comp)
    ref = oracle_select_all(q, k, w.block_size, dens, 1.0, "qk", comp)
    rep = check_selection(sel, ref)
    assert rep["max_stat_err"] < 1e-12, rep


@pytest.mark.parametrize("B,nk,n_tie", [(128, 24, 12), (128, 64, 20), (64, 96, 30)])
def test_topk_exact_ties_take_lower_blocks(ba, B, nk, n_tie):
    """Score ties -> lower g_k (reading A3) with EXACT logit ties: sort='none' keeps the
    blocks contiguous, so n_tie copies of one K block have bit-identical block stats and logits
    on both sides.  The tie group straddles the kappa-th largest in most rows, which runs the
    top-kappa's <= 32-candidate finish (nk 24: from the first radix pass; nk 64 / 96: after the
    passes that isolate the group).  Checked: P4 against the oracle, exact ties in the GPU's
    logits, and in every row the selected members of the group are its lowest-index ones."""
    w = CONFIGS["A"]
    q, k, v = make_qkv(w, device="cuda", seq_len=nk * B, heads_q=2, heads_kv=1)
    rng = np.random.default_rng(nk)
    tie = np.sort(rng.choice(nk, n_tie, replace=False))
    for g in tie[1:]:
        k[:, :, g * B:(g + 1) * B] = k[:, :, tie[0] * B:(tie[0] + 1) * B]
    _, sel = _run_select(ba, q, k, v, B, 0.5, sort="none")
    check_selection(sel, oracle_select_all(q, k, B, 0.5, 1.0, "none", "diag"))
    lg = sel.logits.cpu().numpy()
    assert (lg[..., tie] == lg[..., tie[:1]]).all(), "copies of one key block must tie exactly"
    mask = sel.mask.cpu().numpy().astype(bool)
    partial = 0
    for b_ in range(mask.shape[0]):
        for h in range(mask.shape[1]):
            for g in range(mask.shape[2]):
                chosen = mask[b_, h, g, tie]
                n = int(chosen.sum())
                assert chosen[:n].all() and not chosen[n:].any(), (h, g, chosen)
                partial += 0 < n < n_tie
    assert partial > 0, "no row split the tie group: the case under test did not occur"


@pytest.mark.parametrize("cfg,L,hq,hkv,B", [("A", 4096 + 77, 4, 4, 128), ("C", 8192, 8, 2, 128), ("T", 1024, 1, 1, 64),
                                          ("M", 4096 + 17, 2, 2, 64)])
def test_norm_order_against_exact_norms(ba, cfg, L, hq, hkv, B):
    """S1/S2 checked independently of oracle.norm_key (verdict r1 item 9): the GPU's
    pi must order rows by the EXACT squared norm ||x||^2, computed here
    in fp64 from the very inputs (bf16 / fp32 squares and their 128-term sums are exact or
    within 1e-14 relative in fp64).  The GPU key is an fp32 sum of d products in a fixed
    order: sequential over a lane's d/16 features, then a 4-level tree — at most
    d/16 + 4 + 1 <= 13 roundings, so |key - ||x||^2| <= gamma_13 ||x||^2 (Higham 3.5 with
    gamma_n = n u / (1 - n u), u = 2^-24).  Hence an adjacent pair of pi may be out of
    exact order only when their exact norms differ by at most gamma_13 (a + b)."""
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    ctx, sel = _run_select(ba, q, k, v, B, w.density)
    u = 2.0 ** -24
    gamma = 13 * u / (1 - 13 * u)
    for x, perm in ((q, sel.perm_q), (k, sel.perm_k)):
        xn = x.detach().double().cpu().numpy()
        pn = perm.cpu().numpy()
        for bi in range(xn.shape[0]):
            for h in range(xn.shape[1]):
                exact = (xn[bi, h] * xn[bi, h]).sum(axis=1)
                p = pn[bi, h]
                assert np.array_equal(np.sort(p), np.arange(L)), "pi is not a permutation"
                a, b = exact[p[:-1]], exact[p[1:]]
                bad = (a > b) & (a - b > gamma * (a + b))
                assert not bad.any(), (cfg, h, int(bad.sum()), float((a - b)[bad].max()))
                # identical rows (the synthetic duplicates of T) have identical keys: stable, lower index first
                tie = np.all(xn[bi, h][p[:-1]] == xn[bi, h][p[1:]], axis=1)
                assert (p[:-1][tie] < p[1:][tie]).all()


def test_selection_windowed_and_beta(ba):
    w = CONFIGS["A"]
    q, k, v = make_qkv(w, device="cuda", seq_len=5000, heads_q=2, heads_kv=2)
    _, sel = _run_select(ba, q, k, v, 128, 0.3, beta=0.5, window=1024)
    ref = oracle_select_all(q, k, 128, 0.3, 0.5, "qk", "diag", window=1024)
    check_selection(sel, ref)


def test_selection_batch2(ba):
    w = CONFIGS["C"]
    q, k, v = make_qkv(w, device="cuda", seq_len=2048 + 5, heads_q=4, heads_kv=2, batch=2)
    _, sel = _run_select(ba, q, k, v, 128, 0.5)
    check_selection(sel, oracle_select_all(q, k, 128, 0.5, 1.0, "qk", "diag"))


def test_selection_deterministic(ba):
    w = CONFIGS["A"]
    q, k, v = make_qkv(w, device="cuda", seq_len=4096, heads_q=4, heads_kv=4)
    _, s1 = _run_select(ba, q, k, v, 128, 0.5)
    _, s2 = _run_select(ba, q, k, v, 128, 0.5)
    for f in ("perm_q", "perm_k", "kv_index", "q_sorted", "k_sorted", "v_sorted", "block_prob", "q_mean"):
        assert torch.equal(getattr(s1, f), getattr(s2, f)), f


@pytest.mark.parametrize("cfg,L,hq,hkv,B", [("C", 4096 + 50, 8, 2, 128), ("M", 4096 + 17, 4, 4, 64), ("T", 1024, 1, 1, 64)])
def test_attention_deterministic(ba, cfg, L, hq, hkv, B):
    """SURVEY 8(e) correctness premise: the whole path is deterministic (no
    atomics in any reduction that feeds O), so repeated calls — and therefore
    every rank of a multi-GPU split — reproduce O and LSE bit for bit."""
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    outs = []
    for _ in range(3):
        ctx = ba.Context(q, k, v, B, 0.5)
        ctx.select(q, k, v)
        o = torch.empty_like(q)
        lse = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
        ctx.sparse_attn(o, lse)
        outs.append((o, lse))
    torch.cuda.synchronize()
    for o, lse in outs[1:]:
        assert torch.equal(o, outs[0][0]) and torch.equal(lse, outs[0][1])


# ---------------------------------------------------------------- attention (P5, P6)
def test_attention_fp32_T(ba):
    """Config T end to end: output within 1e-5 of the fp64 oracle."""
    w = CONFIGS["T"]
    q, k, v = make_qkv(w, device="cuda")
    ctx, sel = _run_select(ba, q, k, v, w.block_size, w.density)
    out = torch.empty_like(q)
    ctx.sparse_attn(out)
    torch.cuda.synchronize()
    ref = oracle_output_with_gpu_selection(q, k, v, sel, w.block_size)
    err = max_abs_err(out, ref)
    assert err <= TOL[torch.float32], err
    # and the selection itself matches the oracle's
    check_selection(sel, oracle_select_all(q, k, w.block_size, w.density, 1.0, "qk", "diag"))


def test_attention_fp32_full_density_is_dense(ba):
    w = CONFIGS["T"]
    q, k, v = make_qkv(w, device="cuda")
    out = ba.ba_attention(q, k, v, block_size=64, density=1.0)
    dense = ba.ba_dense_attn(q, k, v, block_size=64)
    torch.cuda.synchronize()
    ref = O.dense_attention(q[0, 0].cpu(), k[0, 0].cpu(), v[0, 0].cpu())
    assert max_abs_err(out[0, 0], ref) <= 1e-5
    assert max_abs_err(dense[0, 0], ref) <= 1e-5


@pytest.mark.parametrize("cfg,L,hq,hkv,dens", [
    ("A", 4096 + 77, 2, 2, 0.5),
    ("C", 4096, 4, 1, 0.25),
    ("V", 2 * 128 * 9 + 80, 2, 2, 0.5),
    ("A", 129, 1, 1, 0.5),
    ("A", 127, 1, 1, 1.0),
    ("A", 1, 1, 1, 1.0),
])
def test_attention_bf16(ba, cfg, L, hq, hkv, dens):
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    ctx, sel = _run_select(ba, q, k, v, w.block_size, dens)
    out = torch.empty_like(q)
    lse = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
    ctx.sparse_attn(out, lse)
    torch.cuda.synchronize()
    ref = oracle_output_with_gpu_selection(q, k, v, sel, w.block_size)
    err = max_abs_err(out, ref)
    assert err <= TOL[torch.bfloat16], err
    assert torch.isfinite(lse).all()


@pytest.mark.parametrize("B,L,hq,hkv", [(128, 2048 + 45, 4, 2), (64, 1024 + 9, 2, 2)])
def test_head_dim_64_bf16(ba, B, L, hq, hkv):
    """head_dim = 64 in bf16 (an ABI combination off the tcgen05 kernels): the
    selection matches the oracle's and the attention matches the oracle run
    with the GPU's selection."""
    w = CONFIGS["A"].with_(head_dim=64, block_size=B)
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    ctx, sel = _run_select(ba, q, k, v, B, 0.5)
    out = torch.empty_like(q)
    ctx.sparse_attn(out)
    torch.cuda.synchronize()
    check_selection(sel, oracle_select_all(q, k, B, 0.5, 1.0, "qk", "diag"))
    err = max_abs_err(out, oracle_output_with_gpu_selection(q, k, v, sel, B))
    assert err <= TOL[torch.bfloat16], err


@pytest.mark.parametrize("L,dens", [(2048 + 33, 0.5), (64 * 31 + 5, 0.3), (64 * 7, 1.0), (100, 0.5)])
def test_attention_bf16_B64(ba, L, dens):
    """B = 64 (dual tiles: two 64-key blocks per 128-key MMA tile), ragged last
    key/query blocks, odd block counts, full density."""
    w = CONFIGS["M"]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=2, heads_kv=2)
    ctx, sel = _run_select(ba, q, k, v, 64, dens)
    out = torch.empty_like(q)
    ctx.sparse_attn(out)
    torch.cuda.synchronize()
    assert max_abs_err(out, oracle_output_with_gpu_selection(q, k, v, sel, 64)) <= 2e-2


def test_bf16_full_density_equals_dense(ba):
    """P6: rho = 1 with sorting on reproduces dense attention (BJ)."""
    w = CONFIGS["A"]
    q, k, v = make_qkv(w, device="cuda", seq_len=1024 + 40, heads_q=2, heads_kv=1)
    out = ba.ba_attention(q, k, v, block_size=128, density=1.0, sort="qk")
    dense = ba.ba_dense_attn(q, k, v)
    torch.cuda.synchronize()
    for h in range(2):
        ref = O.dense_attention(q[0, h].cpu(), k[0, 0].cpu(), v[0, 0].cpu())
        assert max_abs_err(out[0, h], ref) <= 2e-2
        assert max_abs_err(dense[0, h], ref) <= 2e-2


def test_injected_oracle_mask(ba):
    """Kernel-only parity: feed the oracle's permutations and mask through
    ba_sparse_attn (isolates attention from selection)."""
    w = CONFIGS["A"]
    q, k, v = make_qkv(w, device="cuda", seq_len=2048, heads_q=2, heads_kv=2)
    ctx, sel = _run_select(ba, q, k, v, 128, 0.5)
    ref_sel = oracle_select_all(q, k, 128, 0.5, 1.0, "qk", "diag")
    # replace kv_index with a deliberately different (but valid) selection
    rng = np.random.default_rng(3)
    idx = np.sort(np.stack([np.stack([rng.choice(16, 8, replace=False) for _ in range(16)]) for _ in range(2)]), axis=-1)
    sel.kv_index.copy_(torch.from_numpy(idx[None].astype(np.int32)))
    out = torch.empty_like(q)
    ctx.sparse_attn(out)
    torch.cuda.synchronize()
    ref = oracle_output_with_gpu_selection(q, k, v, sel, 128)
    assert max_abs_err(out, ref) <= 2e-2
    assert ref_sel  # oracle selection computed on the same inputs


@pytest.mark.parametrize("B,k5", [(128, "1cta"), (128, "pp"), (128, "pp2"), (64, "dual"), (64, "pair")])
def test_injected_dissimilar_lists(ba, B, k5):
    """Random (dissimilar) index lists for every query block: exercises the
    pair kernels' union walk where a block skips tiles (P = 0 rows), including
    a skipped LAST tile (the epilogue must still wait for every PV), and for
    B = 64 odd union lengths (the dual kernel's half-empty last tile)."""
    import subprocess, sys, os
    env = dict(os.environ, **({"BA_ATTN_K5": k5} if B == 128 else {"BA_ATTN_B64": k5}))
    code = f"""
import sys; sys.path.insert(0, {os.path.join(os.path.dirname(__file__))!r}); sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import numpy as np, torch
import paper_2605_19726_b200.baatt as ba
from synth import CONFIGS, make_qkv
from parity import oracle_output_with_gpu_selection, max_abs_err
B = {B}
w = CONFIGS["A" if B == 128 else "M"]
for seed in range(4):
    q, k, v = make_qkv(w, device="cuda", seq_len=16 * B + 37, heads_q=2, heads_kv=1)
    ctx = ba.Context(q, k, v, B, 0.5)
    sel = ctx.select(q, k, v)
    nk, kap = sel.n_k, sel.kappa
    rng = np.random.default_rng(seed)
    idx = np.sort(np.stack([np.stack([rng.choice(nk, kap, replace=False) for _ in range(sel.n_q)]) for _ in range(2)]), axis=-1)
    sel.kv_index.copy_(torch.from_numpy(idx[None].astype(np.int32)))
    out = torch.empty_like(q)
    ctx.sparse_attn(out)
    torch.cuda.synchronize()
    err = max_abs_err(out, oracle_output_with_gpu_selection(q, k, v, sel, B))
    assert err <= 2e-2, (seed, err)
print("OK", ba.attention_kernel_name(q, k, v, B))
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=240)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("B", [128, 64])
def test_running_max_grows_every_tile(ba, B):
    """B = 128 pair kernel / B = 64 dual-tile kernel: key scale grows along the sequence, so in
    ba_dense_attn (no permutation, key blocks walked in ascending order) the row max
    of every tile exceeds the running max by far more than the lazy-rescale threshold
    (2^8): every tile takes the rescale path, and with the speculative row max the
    first P part is recomputed on every tile.  LSE checks the running max / sum."""
    torch.manual_seed(11)
    L, d, hq = 128 * 12 + 41, 128, 2
    q = torch.randn(1, hq, L, d)
    q[:, 1] *= -1.0  # the second head sees shrinking maxima along the walk (no rescale)
    # key scale grows linearly: a row's tile max grows by ~7 nats (~10 log2 units) per key block
    growth = 2.0 + 2.5 * torch.arange(L, dtype=torch.float32) / 128
    k = (torch.randn(1, 1, L, d).abs() + 0.5) * growth[None, None, :, None]
    v = torch.randn(1, 1, L, d)
    q, k, v = (t.to(torch.bfloat16).cuda() for t in (q, k, v))
    lse = torch.empty(1, hq, L, dtype=torch.float32, device="cuda")
    out = ba.ba_dense_attn(q, k, v, lse=lse, block_size=B)
    torch.cuda.synchronize()
    scale = 1.0 / math.sqrt(d)
    for h in range(hq):
        qh, kh, vh = (t.double().cpu().numpy() for t in (q[0, h], k[0, 0], v[0, 0]))
        ref = O.dense_attention(qh, kh, vh)
        assert max_abs_err(out[0, h], ref) <= 2e-2, h
        s = qh @ kh.T * scale
        mx = s.max(axis=1)
        ref_lse = mx + np.log(np.exp(s - mx[:, None]).sum(axis=1))
        err = np.abs(lse[0, h].cpu().numpy() - ref_lse) / np.maximum(1.0, np.abs(ref_lse))
        assert err.max() <= 1e-3, (h, float(err.max()))


def test_pp_scatter4_epilogue_bitwise(ba):
    """NEXT-2 un-permute by TMA tile::scatter4 (dense O, full 128-row blocks) is bit-identical
    to per-thread row stores (BA_PP_SCATTER=0), including the ragged last block (always
    per-thread) and LSE, and both match the oracle."""
    import os, subprocess, sys
    code = f"""
import sys; sys.path.insert(0, {os.path.dirname(__file__)!r}); sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import torch
import paper_2605_19726_b200.baatt as ba
from synth import CONFIGS, make_qkv
w = CONFIGS["C"]
q, k, v = make_qkv(w, device="cuda", seq_len=128 * 13 + 57, heads_q=4, heads_kv=1, batch=2)
ctx = ba.Context(q, k, v, 128, 0.5)
ctx.select(q, k, v)
out = torch.empty_like(q)
lse = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
ctx.sparse_attn(out, lse)
torch.cuda.synchronize()
torch.save((out.cpu(), lse.cpu()), sys.argv[1])
print("OK", ba.attention_kernel_name(q, k, v, 128))
"""
    outs = []
    for env_val in ("1", "0"):
        path = f"/tmp/ba_scatter_{env_val}.pt"
        env = dict(os.environ, BA_PP_SCATTER=env_val)
        r = subprocess.run([sys.executable, "-c", code, path], capture_output=True, text=True, env=env, timeout=240)
        assert r.returncode == 0 and "OK attn_sm100_tcgen05_pp" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
        outs.append(torch.load(path))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_pp_unequal_lists_split_steps(ba):
    """Injected lists of unequal lengths (kv_count) with disjoint halves: the pair
    kernel's walk runs shared tiles, split tiles (A and B on different key blocks) and
    a one-sided tail (P = 0 for the block that ran out), with the ragged last key
    block landing on each kind of step."""
    w = CONFIGS["A"]
    for seed in range(3):
        q, k, v = make_qkv(w, device="cuda", seq_len=128 * 14 + 29, heads_q=2, heads_kv=1)
        ctx = ba.Context(q, k, v, 128, 0.5)
        sel = ctx.select(q, k, v)
        nk, kap, nq = sel.n_k, sel.kappa, sel.n_q
        rng = np.random.default_rng(100 + seed)
        idx = np.zeros((2, nq, kap), np.int32)
        cnt = np.zeros((2, nq), np.int32)
        for h in range(2):
            for g in range(nq):
                c = int(rng.integers(1, kap + 1))
                pick = np.sort(rng.choice(nk, c, replace=False))
                if g % 3 == 0 and (nk - 1) not in pick:
                    pick[-1] = nk - 1  # the ragged block on a split or one-sided step
                    pick = np.unique(pick)
                idx[h, g, :len(pick)] = pick
                idx[h, g, len(pick):] = pick[-1]
                cnt[h, g] = len(pick)
        sel.kv_index.copy_(torch.from_numpy(idx[None]))
        sel.kv_count.copy_(torch.from_numpy(cnt[None]))
        out = torch.empty_like(q)
        ctx.sparse_attn(out)
        torch.cuda.synchronize()
        err = max_abs_err(out, oracle_output_with_gpu_selection(q, k, v, sel, 128))
        assert err <= 2e-2, (seed, err)


@pytest.mark.parametrize("cfg,L,hq,hkv,b", [("A", 1024, 2, 2, 1), ("C", 2048 + 64, 8, 2, 2), ("A", 1000, 16, 16, 1)])
def test_end_to_end_host_api(ba, cfg, L, hq, hkv, b):
    """ba_attention_host (chunked over KV heads, copies overlapped with compute)
    is bit-identical to ba_attention on device-resident inputs."""
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cpu", seq_len=L, heads_q=hq, heads_kv=hkv, batch=b)
    qh, kh, vh = q.pin_memory(), k.pin_memory(), v.pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    ws = torch.empty(ba.attention_host_workspace_size(qh, kh, vh), dtype=torch.uint8, device="cuda")
    ba.ba_attention_host(qh, kh, vh, oh, ws)
    torch.cuda.synchronize()
    dev = ba.ba_attention(q.cuda(), k.cuda(), v.cuda())
    torch.cuda.synchronize()
    assert torch.equal(oh, dev.cpu())


def test_errors_are_loud(ba):
    w = CONFIGS["A"]
    q, k, v = make_qkv(w, device="cuda", seq_len=256, heads_q=3, heads_kv=2)
    with pytest.raises(ba.BaError, match="SHAPE_MISMATCH"):
        ba.ba_attention(q, k, v)


@pytest.mark.parametrize("k5,name", [("pp", "attn_sm100_tcgen05_pp"), ("pp2", "attn_sm100_tcgen05_pp2"),
                                     ("1cta", "attn_sm100_tcgen05")])
def test_b128_kernel_parity(ba, k5, name):
    """Each B = 128 kernel (BA_ATTN_K5 = pp | 1cta) on real selections,
    ragged lengths, GQA and an odd number of query blocks."""
    import os, subprocess, sys
    env = dict(os.environ, BA_ATTN_K5=k5)
    code = f"""
import sys; sys.path.insert(0, {os.path.dirname(__file__)!r}); sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import torch
import paper_2605_19726_b200.baatt as ba
from synth import CONFIGS, make_qkv
from parity import oracle_output_with_gpu_selection, max_abs_err
for cfg, L, hq, hkv, dens in (("A", 4096 + 77, 2, 2, 0.5), ("C", 3 * 128 * 5, 4, 1, 0.25), ("V", 2 * 128 * 9 + 80, 2, 2, 0.5)):
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    ctx = ba.Context(q, k, v, 128, dens)
    sel = ctx.select(q, k, v)
    out = torch.empty_like(q)
    ctx.sparse_attn(out)
    torch.cuda.synchronize()
    err = max_abs_err(out, oracle_output_with_gpu_selection(q, k, v, sel, 128))
    assert err <= 2e-2, (cfg, err)
print("OK", ba.attention_kernel_name(q, k, v, 128))
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=240)
    assert r.returncode == 0 and f"OK {name}\n" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("k5,name", [("dual", "attn_sm100_tcgen05_dual64")])
def test_b64_kernel_parity(ba, k5, name):
    """The B = 64 dual-tile kernel on real selections: ragged lengths (a ragged last
    key block), odd query- and key-block counts (a half-empty last tile), GQA, top-p
    lists of unequal length, and the per-tile rescale workload (key scale growing
    along the sequence, dense) that exercises the speculative row max's redo."""
    import os, subprocess, sys
    env = dict(os.environ, BA_ATTN_B64=k5)
    code = f"""
import sys, math; sys.path.insert(0, {os.path.dirname(__file__)!r}); sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import numpy as np, torch
import oracle as O
import paper_2605_19726_b200.baatt as ba
from synth import CONFIGS, make_qkv
from parity import oracle_output_with_gpu_selection, max_abs_err
for cfg, L, hq, hkv, dens, top_p in (("M", 64 * 37 + 5, 2, 2, 0.5, None), ("M", 64 * 21, 4, 2, 0.3, None),
                                     ("M", 64 * 30 + 63, 2, 1, 0.5, 0.9), ("M", 64 * 9, 1, 1, 1.0, None)):
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    ctx = ba.Context(q, k, v, 64, dens, top_p=top_p)
    sel = ctx.select(q, k, v)
    out = torch.empty_like(q)
    ctx.sparse_attn(out)
    torch.cuda.synchronize()
    err = max_abs_err(out, oracle_output_with_gpu_selection(q, k, v, sel, 64))
    assert err <= 2e-2, (cfg, L, err)
torch.manual_seed(5)
L = 64 * 19 + 23
q = torch.randn(1, 2, L, 128); q[:, 1] *= -1.0
k = (torch.randn(1, 1, L, 128).abs() + 0.5) * (2.0 + 1.25 * torch.arange(L, dtype=torch.float32) / 64)[None, None, :, None]
v = torch.randn(1, 1, L, 128)
q, k, v = (t.to(torch.bfloat16).cuda() for t in (q, k, v))
out = ba.ba_dense_attn(q, k, v, block_size=64)
torch.cuda.synchronize()
for h in range(2):
    ref = O.dense_attention(q[0, h].double().cpu().numpy(), k[0, 0].double().cpu().numpy(), v[0, 0].double().cpu().numpy())
    assert max_abs_err(out[0, h], ref) <= 2e-2, ("rescale", h)
print("OK", ba.attention_kernel_name(q, k, v, 64))
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0 and f"OK {name}\n" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


# ---------------------------------------------------------------- NEXT-1: cumulative-mass budget (reading A23)
@pytest.mark.parametrize("cfg,L,hq,hkv,B,dens,top_p", [
    ("T", 1024, 1, 1, 64, 1.0, 0.9),
    ("A", 4096 + 77, 4, 4, 128, 1.0, 0.5),
    ("C", 8192, 8, 2, 128, 0.5, 0.95),    # cap binds on flat rows
    ("M", 4096 + 13, 2, 2, 64, 1.0, 0.99),
    ("V", 4500, 2, 2, 128, 0.4, 0.7),
])
def test_selection_topp(ba, cfg, L, hq, hkv, B, dens, top_p):
    """TOPP masks and kappa_row vs the oracle (P4 with the cumulative-mass band),
    then the attention over the variable-length lists (P5)."""
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    p32 = float(np.float32(top_p))  # the ABI carries top_p as fp32
    ctx = ba.Context(q, k, v, B, dens, diagnostics=True, top_p=p32)
    sel = ctx.select(q, k, v)
    out = torch.empty_like(q)
    ctx.sparse_attn(out)
    torch.cuda.synchronize()
    ref = oracle_select_all(q, k, B, dens, 1.0, "qk", "diag", top_p=p32)
    check_selection(sel, ref)
    cnt = sel.kv_count.cpu().numpy()
    assert (cnt >= 1).all() and (cnt <= sel.kappa).all()
    tol = TOL[q.dtype]
    assert max_abs_err(out, oracle_output_with_gpu_selection(q, k, v, sel, B)) <= tol


def test_topp_full_mass_keeps_everything(ba):
    """top_p = 1 with density 1: every row whose mass sums below 1 in fp64
    keeps all N_k blocks; the rest keep the prefix that reaches 1 — either way
    the oracle's kappa_row (checked by check_selection)."""
    w = CONFIGS["A"]
    q, k, v = make_qkv(w, device="cuda", seq_len=2048, heads_q=2, heads_kv=2)
    ctx = ba.Context(q, k, v, 128, 1.0, diagnostics=True, top_p=1.0)
    sel = ctx.select(q, k, v)
    torch.cuda.synchronize()
    check_selection(sel, oracle_select_all(q, k, 128, 1.0, 1.0, "qk", "diag", top_p=1.0))


def test_topp_rejects_bad_p(ba):
    w = CONFIGS["A"]
    q, k, v = make_qkv(w, device="cuda", seq_len=256, heads_q=1, heads_kv=1)
    for bad in (0.0, 1.5, -0.1):
        with pytest.raises(ba.BaError, match="INVALID_ARGUMENT"):
            ba.Context(q, k, v, 128, 0.5, top_p=bad).select(q, k, v)


# ---------------------------------------------------------------- NEXT-2: zero-copy permutation (TMA gather4)
@pytest.mark.parametrize("cfg,L,hq,hkv,B,dens,b", [
    ("A", 4096 + 77, 2, 2, 128, 0.5, 1),   # ragged last key / query block
    ("C", 3 * 128 * 5, 4, 1, 128, 0.25, 2),  # GQA, batch 2, odd block count
    ("V", 2 * 128 * 9 + 80, 2, 2, 128, 0.5, 1),
    ("M", 2048 + 33, 2, 2, 64, 0.5, 1),    # B = 64 dual tiles
    ("M", 64 * 31 + 5, 2, 1, 64, 0.3, 1),
])
@pytest.mark.parametrize("k5", ["pp", "1cta"])
def test_zero_copy_matches_copies(ba, cfg, L, hq, hkv, B, dens, b, k5):
    """ba_sparse_attn_gather (rows fetched through pi_q / pi_k by TMA gather4,
    no Q'/K'/V' copies) is bit-identical to ba_sparse_attn on the permuted
    copies, and within the bf16 tolerance of the oracle (P5)."""
    import os, subprocess, sys
    code = f"""
import sys; sys.path.insert(0, {os.path.dirname(__file__)!r}); sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import torch
import paper_2605_19726_b200.baatt as ba
from synth import CONFIGS, make_qkv
from parity import oracle_output_with_gpu_selection, max_abs_err
w = CONFIGS[{cfg!r}]
q, k, v = make_qkv(w, device="cuda", seq_len={L}, heads_q={hq}, heads_kv={hkv}, batch={b})
assert ba.zero_copy_supported(q, k, v, {B})
c0 = ba.Context(q, k, v, {B}, {dens})
c1 = ba.Context(q, k, v, {B}, {dens}, zero_copy=True)
c3 = ba.Context(q, k, v, {B}, {dens}, zero_copy="q")
s0 = c0.select(q, k, v); s1 = c1.select(q, k, v); s3 = c3.select(q, k, v)
assert s1.q_sorted is None and s1.v_sorted is None
assert s3.q_sorted is None and s3.k_sorted is not None
o0 = torch.empty_like(q); o1 = torch.full_like(q, float("nan")); o3 = torch.full_like(q, float("nan"))
c0.sparse_attn(o0); c1.sparse_attn(o1); c3.sparse_attn(o3)
assert torch.equal(o0, o3)
assert torch.equal(s0.k_sorted, s3.k_sorted) and torch.equal(s0.v_sorted, s3.v_sorted)
o2 = ba.ba_attention(q, k, v, block_size={B}, density={dens})  # copy path
torch.cuda.synchronize()
for f in ("perm_q", "perm_k", "kv_index", "kv_count"):
    assert torch.equal(getattr(s0, f), getattr(s1, f)), f
assert torch.equal(o0, o1), (o0.float() - o1.float()).abs().max().item()
assert torch.equal(o0, o2)
err = max_abs_err(o1, oracle_output_with_gpu_selection(q, k, v, s1, {B}))
assert err <= 2e-2, err
print("OK", ba.attention_kernel_name(q, k, v, {B}))
"""
    for zc in ("0", "1", "2"):  # ba_attention: copies / BA_ZERO_COPY=1 (none) / =2 (Q in place)
        env = dict(os.environ, BA_ATTN_K5=k5, BA_ZERO_COPY=zc)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
        assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_zero_copy_unsupported_layout_falls_back_to_copies(ba):
    """A non-dense (b, h) layout is not zero-copy eligible: ba_sparse_attn_gather
    refuses it loudly and ba_attention takes the permuted-copy path."""
    w = CONFIGS["A"]
    q, k, v = make_qkv(w, device="cuda", seq_len=1024, heads_q=2, heads_kv=2)
    big = torch.zeros(1, 4, 1024, 128, dtype=q.dtype, device="cuda")
    big[:, ::2] = q
    qs = big[:, ::2]  # head stride 2*L*d != L*d: rows are not one (b*H*L, d) row space
    assert not ba.zero_copy_supported(qs, k, v, 128)
    with pytest.raises(ba.BaError, match="UNSUPPORTED"):
        ba.Context(qs, k, v, 128, 0.5, zero_copy=True)
    out = ba.ba_attention(qs, k, v)
    ref = ba.ba_attention(q, k, v)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


# ---------------------------------------------------------------- NEXT-4: exact covariance compensation
@pytest.mark.parametrize("cfg,L,hq,hkv,B,dens,beta", [
    ("T", 1024, 1, 1, 64, 0.5, 1.0),          # fp32, d = 64
    ("A", 2048 + 77, 2, 2, 128, 0.5, 1.0),    # ragged last block
    ("C", 1024 * 3, 4, 1, 128, 0.25, 0.5),    # GQA, beta != 1
    ("M", 1024 + 13, 2, 2, 64, 0.5, 1.0),
])
def test_selection_exact_compensation(ba, cfg, L, hq, hkv, B, dens, beta):
    """BA_COMP_EXACT: Delta = tr(SigmaQ SigmaK)/d from full per-block covariances
    (Eq. cov-comp) — masks within the band of the oracle's
    compensation_exact selection, m' within 1e-12, outputs within tolerance."""
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    ctx = ba.Context(q, k, v, B, dens, beta, "qk", "exact", diagnostics=True)
    sel = ctx.select(q, k, v)
    out = torch.empty_like(q)
    ctx.sparse_attn(out)
    torch.cuda.synchronize()
    ref = oracle_select_all(q, k, B, dens, beta, "qk", "exact")
    rep = check_selection(sel, ref)
    assert rep["max_abs_dm"] < 1e-12, rep
    # and the exact rule differs from the diagonal one somewhere (the test is not vacuous)
    diag = oracle_select_all(q, k, B, dens, beta, "qk", "diag")
    assert any(np.abs(ref[kk].m - diag[kk].m).max() > 1e-9 for kk in ref)
    assert max_abs_err(out, oracle_output_with_gpu_selection(q, k, v, sel, B)) <= TOL[q.dtype]


# ---------------------------------------------------------------- NEXT-3: oracle block distribution on the GPU
@pytest.mark.parametrize("cfg,L,hq,hkv,dens", [("A", 2048 + 77, 2, 2, 0.5), ("C", 1024 * 3, 4, 1, 0.25), ("V", 128 * 9 + 80, 2, 2, 0.5)])
def test_block_mass_matches_oracle(ba, cfg, L, hq, hkv, dens):
    """ba_block_mass: m_hat (Eq. oracle-dist) of the dense softmax in the
    sorted block space vs the fp64 oracle's oracle_block_mass(dense map), and the
    selection's captured mass.  Tolerance: S is an fp32 sum of exact bf16 products
    (relative error ~1e-6 |S|), exp2 / LSE in fp32: |dm_hat| <= 3e-5 + 1e-3 m_hat."""
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    ctx = ba.Context(q, k, v, 128, dens)
    sel = ctx.select(q, k, v)
    m_hat, cap = ctx.block_mass()
    torch.cuda.synchronize()
    mh = m_hat.double().cpu().numpy()
    cp = cap.double().cpu().numpy()
    pq, pk, idx, cnt = (sel.perm_q.cpu().numpy(), sel.perm_k.cpu().numpy(), sel.kv_index.cpu().numpy(),
                        sel.kv_count.cpu().numpy())
    grp = hq // hkv
    for h in range(hq):
        Qs = O.apply_permutation(q[0, h].cpu(), pq[0, h])
        Ks = O.apply_permutation(k[0, h // grp].cpu(), pk[0, h // grp])
        ref = O.oracle_block_mass(O.dense_attention_map(Qs, Ks), 128, 128)
        np.testing.assert_allclose(mh[0, h], ref, atol=3e-5, rtol=1e-3)
        np.testing.assert_allclose(mh[0, h].sum(1), 1.0, atol=1e-4)
        ref_cap = np.array([ref[g, idx[0, h, g, :cnt[0, h, g]]].sum() for g in range(ref.shape[0])])
        np.testing.assert_allclose(cp[0, h], ref_cap, atol=1e-4, rtol=1e-3)


def test_block_mass_fullsize_properties(ba):
    """Config A, one head at full length (32K): rows of m_hat sum to 1, the
    selection's captured mass never exceeds the greedy optimum (top-kappa of
    m_hat itself), and the selection captures more mass than kappa
    blocks chosen at random would on average (kappa / N_k)."""
    w = CONFIGS["A"]
    q, k, v = make_qkv(w, device="cuda", heads_q=1, heads_kv=1)
    ctx = ba.Context(q, k, v, 128, 0.5)
    sel = ctx.select(q, k, v)
    m_hat, cap = ctx.block_mass()
    torch.cuda.synchronize()
    mh = m_hat[0, 0].double()
    assert torch.allclose(mh.sum(1), torch.ones_like(mh[:, 0]), atol=1e-3)
    kap = sel.kappa
    greedy = torch.topk(mh, kap, dim=1).values.sum(1)
    c = cap[0, 0].double()
    assert (c <= greedy + 1e-4).all()
    assert c.mean() > kap / sel.n_k + 0.05


# ---------------------------------------------------------------- fused output collective (peer stores)
@pytest.mark.parametrize("cfg,L,hq,hkv,B", [("C", 2048 + 64, 4, 1, 128), ("M", 2048 + 33, 2, 2, 64)])
def test_sparse_attn_peers_broadcast(ba, cfg, L, hq, hkv, B):
    """ba_sparse_attn_peers stores every output row to each peer buffer (here
    three buffers of one device, slices of a larger 'full' buffer as a
    head-parallel rank would see them): each copy equals ba_sparse_attn."""
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    ref = torch.empty_like(q)
    ctx0 = ba.Context(q, k, v, B, 0.5)
    ctx0.select(q, k, v)
    ctx0.sparse_attn(ref)
    # full buffers of 2*hq heads; this "rank" owns heads [hq, 2*hq)
    fulls = [torch.full((1, 2 * hq, L, 128), float("nan"), dtype=q.dtype, device="cuda") for _ in range(3)]
    from paper_2605_19726_b200.dist import peer_slice_ptrs
    ptrs = peer_slice_ptrs([f.data_ptr() for f in fulls], hq, fulls[0].stride(1), 2)
    ctx = ba.Context(q, k, v, B, 0.5, out=fulls[0][:, hq:])
    ctx.select(q, k, v)
    ctx.sparse_attn_peers(ptrs)
    torch.cuda.synchronize()
    for f in fulls:
        assert torch.equal(f[:, hq:], ref)
        assert torch.isnan(f[:, :hq].float()).all()  # nothing written outside this rank's heads


# ---------------------------------------------------------------- uneven split: work units
@pytest.mark.parametrize("cfg,L,hq,hkv,B", [("C", 2048 + 64, 8, 2, 128), ("M", 2048 + 33, 5, 5, 64),
                                            ("T", 1000, 3, 3, 64)])
@pytest.mark.parametrize("world", [3, 8])
def test_sparse_attn_units_reassemble_bitwise(ba, cfg, L, hq, hkv, B, world):
    """Each simulated rank selects over the heads its units touch (whole GQA
    groups) and runs ba_sparse_attn_units on its unit range; the union of the
    ranks' rows is the 1-GPU ba_sparse_attn output and LSE, bit for bit."""
    from paper_2605_19726_b200.dist import unit_heads, unit_range
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    ref, lse_ref = torch.empty_like(q), torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
    ctx0 = ba.Context(q, k, v, B, 0.5)
    ctx0.select(q, k, v)
    ctx0.sparse_attn(ref, lse_ref)
    nq = ctx0.sel.n_q
    out = torch.full_like(q, float("nan"))
    lse = torch.full_like(lse_ref, float("nan"))
    for r in range(world):
        u0, u1 = unit_range(hq, nq, world, r)
        q0, q1, k0, k1 = unit_heads(u0, u1, nq, hq, hkv)
        if u1 <= u0:
            continue
        qs, ks, vs = q[:, q0:q1].contiguous(), k[:, k0:k1].contiguous(), v[:, k0:k1].contiguous()
        ctx = ba.Context(qs, ks, vs, B, 0.5, out=out[:, q0:q1])
        ctx.select(qs, ks, vs)
        ctx.sparse_attn_units(u0 - q0 * nq, u1 - q0 * nq, [out[:, q0:q1]], lse=lse[:, q0:q1])
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    assert torch.equal(lse, lse_ref)


def test_sparse_attn_units_batch_and_peers(ba):
    """Unit ranges crossing head and batch boundaries of one selection (b = 2,
    GQA) cover the output exactly once; with two outputs every row lands in
    both (the peer-store path)."""
    w = CONFIGS["C"]
    B, L, hq, hkv = 128, 1536 + 40, 4, 2
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv, batch=2)
    ref = torch.empty_like(q)
    ctx = ba.Context(q, k, v, B, 0.5)
    ctx.select(q, k, v)
    ctx.sparse_attn(ref)
    nq = ctx.sel.n_q
    n = 2 * hq * nq
    cuts = [0, 5, nq, nq + 1, 3 * nq - 2, 5 * nq + 3, n]
    outs = [torch.full_like(q, float("nan")) for _ in range(2)]
    for a, b_ in zip(cuts[:-1], cuts[1:]):
        ctx.sparse_attn_units(a, b_, outs[:1])
    torch.cuda.synchronize()
    assert torch.equal(outs[0], ref)
    outs[0].fill_(float("nan"))
    for a, b_ in zip(cuts[:-1], cuts[1:]):
        ctx.sparse_attn_units(a, b_, outs)
    ctx.sparse_attn_units(n, n, outs)  # empty range: nothing enqueued
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)
    with pytest.raises(ba.BaError):
        ctx.sparse_attn_units(0, n + 1, outs[:1])


def test_fused_head_gather_symmetric_memory(tmp_path):
    """The fused output collective end to end on one rank under torchrun: NCCL
    process group, a symmetric-memory full O (torch symm_mem rendezvous), the
    attention epilogue storing through the peer pointers (ba_sparse_attn_peers,
    and ba_sparse_attn_units for a unit split), then the symmetric barrier —
    equal to ba_sparse_attn bit for bit."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "fused.py"
    script.write_text(f"""
import sys; sys.path.insert(0, {root!r}); sys.path.insert(0, {os.path.dirname(os.path.abspath(__file__))!r})
import torch, torch.distributed as dist
import paper_2605_19726_b200.baatt as ba
from paper_2605_19726_b200.dist import FusedHeadGather
from synth import CONFIGS, make_qkv
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
w = CONFIGS["C"]
q, k, v = make_qkv(w, device=dev, seq_len=2048 + 64, heads_q=8, heads_kv=2)
ref = torch.empty_like(q)
c0 = ba.Context(q, k, v, 128, 0.5)
c0.select(q, k, v)
c0.sparse_attn(ref)
f = FusedHeadGather(tuple(q.shape), q.dtype, dev, 0)
f.full.fill_(float("nan"))
ctx = ba.Context(q, k, v, 128, 0.5, out=f.full)
ctx.select(q, k, v)
ctx.sparse_attn_peers(f.peer_ptrs)
f.barrier()
torch.cuda.synchronize()
ok1 = torch.equal(f.full, ref)
f.full.fill_(float("nan"))
n = 8 * ctx.sel.n_q
ctx.sparse_attn_units(0, n // 3, f.peer_ptrs)
ctx.sparse_attn_units(n // 3, n, f.peer_ptrs)
f.barrier()
torch.cuda.synchronize()
ok2 = torch.equal(f.full, ref)
mc = "unavailable"
if f.mc_ptr:  # NVLS multicast stores (ba_sparse_attn_multicast), when the system supports multicast
    f.full.fill_(float("nan"))
    ctx.sparse_attn_multicast(f.mc_ptr)
    f.barrier()
    torch.cuda.synchronize()
    mc = str(torch.equal(f.full, ref))
dist.destroy_process_group()
print("MULTICAST", mc)
print("RESULT", ok1, ok2, mc != "False")
""")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", "29561", str(script)],
                       capture_output=True, text=True, timeout=300, cwd=root)
    assert "RESULT True True True" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


# ---------------------------------------------------------------- boundary: S:393 empty rows, bad indices
@pytest.mark.parametrize("cfg,B,k5", [("A", 128, "pp"), ("A", 128, "pp2"), ("A", 128, "1cta"), ("M", 64, "dual"),
                                      ("T", 64, "simt")])
def test_empty_mask_row_is_reported(ba, cfg, B, k5):
    """An injected kv_count = 0 violates the non-empty-row precondition:
    the kernels write those rows as O = 0, LSE = -inf (never unwritten TMEM),
    leave every other row as computed, and ba_check_errors reports
    BA_ERR_EMPTY_MASK_ROW (once: the latch clears).  Both blocks of a pair empty
    (no MMA at all in the pair CTA) and one of a pair empty are covered."""
    import os, subprocess, sys
    env = dict(os.environ, BA_ATTN_K5=k5 if B == 128 else "pp")
    code = f"""
import sys; sys.path.insert(0, {os.path.dirname(__file__)!r}); sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import torch
import paper_2605_19726_b200.baatt as ba
from synth import CONFIGS, make_qkv
from parity import oracle_output_with_gpu_selection, max_abs_err
B = {B}
w = CONFIGS[{cfg!r}]
q, k, v = make_qkv(w, device="cuda", seq_len=12 * B + 5, heads_q=2, heads_kv=1 if w.heads_kv != w.heads_q else 2)
ctx = ba.Context(q, k, v, B, 0.5)
sel = ctx.select(q, k, v)
torch.cuda.synchronize()
ba.ba_check_errors()  # clean
empty = [(0, 0), (0, 1), (1, 3), (1, 12)]  # head 0: both blocks of pair 0; head 1: one block of a pair; last block
for h, g in empty:
    sel.kv_count[0, h, g] = 0
out = torch.full_like(q, 7.0)
lse = torch.zeros(q.shape[:3], dtype=torch.float32, device="cuda")
ctx.sparse_attn(out, lse)
try:
    ba.ba_check_errors()
    raise SystemExit("no error latched")
except ba.BaError as e:
    assert "EMPTY_MASK_ROW" in str(e), e
ba.ba_check_errors()  # the latch cleared
perm = sel.perm_q[0].long()
for h, g in empty:
    rows = perm[h, g * B:min(q.shape[2], (g + 1) * B)]
    assert torch.all(out[0, h, rows] == 0), (h, g)
    assert torch.all(torch.isneginf(lse[0, h, rows])), (h, g)
# every other row as the oracle computes it (rows of unrequested blocks are NaN there and skipped)
qb = {{(0, h): [g for g in range(sel.n_q) if (h, g) not in empty] for h in range(2)}}
ref = oracle_output_with_gpu_selection(q, k, v, sel, B, q_blocks=qb)
err = max_abs_err(out, ref)
assert err <= (1e-5 if q.dtype == torch.float32 else 2e-2), err
# an out-of-range index is skipped and reported as an invalid argument
sel.kv_count.fill_(sel.kappa)
sel.kv_index[0, 0, 2, 0] = sel.n_k + 5
ctx.sparse_attn(out)
try:
    ba.ba_check_errors()
    raise SystemExit("no error latched")
except ba.BaError as e:
    assert "INVALID_ARGUMENT" in str(e), e
print("OK", ba.attention_kernel_name(q, k, v, B))
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=240)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_context_tracks_latest_inputs_and_checks_layouts(ba):
    """ADVICE fixes: a Context reused on new activations runs the zero-copy
    attention on the tensors of the LATEST select() (not the construction-time
    ones), equal to the copy path on those tensors; mismatched input / output
    layouts and injected selections of another kappa raise instead of being
    written with the wrong strides."""
    w = CONFIGS["A"]
    q, k, v = make_qkv(w, device="cuda", seq_len=1024 + 64, heads_q=2, heads_kv=2)
    q2, k2, v2 = make_qkv(w.with_(config_index=77), device="cuda", seq_len=1024 + 64, heads_q=2, heads_kv=2)
    zc = ba.Context(q, k, v, 128, 0.5, zero_copy=True)
    cp = ba.Context(q2, k2, v2, 128, 0.5)
    zc.select(q, k, v)
    zc.select(q2, k2, v2)
    o_zc, o_cp = torch.empty_like(q), torch.empty_like(q)
    zc.sparse_attn(o_zc)
    cp.select(q2, k2, v2)
    cp.sparse_attn(o_cp)
    torch.cuda.synchronize()
    assert torch.equal(o_zc, o_cp)
    with pytest.raises(ba.BaError, match="SHAPE_MISMATCH"):
        zc.select(q2[:, :1].contiguous(), k2, v2)
    bad = torch.empty(q.shape[0], q.shape[2], q.shape[1], q.shape[3], dtype=q.dtype, device="cuda").transpose(1, 2)
    with pytest.raises(ba.BaError, match="SHAPE_MISMATCH"):
        cp.sparse_attn(bad)
    other = ba.Context(q, k, v, 128, 0.25).select(q, k, v)
    with pytest.raises(ba.BaError, match="SHAPE_MISMATCH"):
        cp.sparse_attn(o_cp, sel=other)
    with pytest.raises(ba.BaError, match="SHAPE_MISMATCH"):
        ba.ba_sparse_attn(q, k, v, other, density=0.5)
    out = ba.ba_sparse_attn(q, k, v, other)  # density derived from the selection's kappa
    ref = ba.Context(q, k, v, 128, 0.25)
    ref.select(q, k, v)
    o_ref = torch.empty_like(q)
    ref.sparse_attn(o_ref)
    torch.cuda.synchronize()
    assert torch.equal(out, o_ref)


# ---------------------------------------------------------------- NEXT-3: bound U and observed max deviation
@pytest.mark.parametrize("cfg,L,hq,hkv,sort", [("A", 1024 + 77, 2, 2, "qk"), ("C", 2048, 4, 1, "qk"),
                                               ("V", 1500, 2, 2, "none"), ("A", 640, 1, 1, "q")])
def test_deviation_bound_matches_oracle(ba, cfg, L, hq, hkv, sort):
    """ba_deviation vs the oracle on the GPU's sorted copies: U (Eq. logits-bound,
    P:376-383) to 1e-10 relative (fp64 on both sides), the observed
    max |l_hat - l| (Fig. 2) within the fp32-accumulation bound
    d*2^-24*M^Q M^K/sqrt(d) + 1e-9, and U >= max_dev on every block pair (the
    theorem, up to that rounding)."""
    w = CONFIGS[cfg]
    q, k, v = make_qkv(w, device="cuda", seq_len=L, heads_q=hq, heads_kv=hkv)
    ctx = ba.Context(q, k, v, 128, 0.5, sort=sort, diagnostics=True)
    sel = ctx.select(q, k, v)
    U, dev = ctx.deviation()
    torch.cuda.synchronize()
    grp = hq // hkv
    for h in range(hq):
        Qs = sel.q_sorted[0, h].float().cpu().numpy()
        Ks = sel.k_sorted[0, h // grp].float().cpu().numpy()
        U_ref = O.deviation_bound(Qs, Ks, 128)
        dev_ref = O.max_logit_deviation(Qs, Ks, 128)
        Ug, dg = U[0, h].cpu().numpy(), dev[0, h].cpu().numpy()
        assert np.abs(Ug - U_ref).max() <= 1e-10 * (1 + np.abs(U_ref).max())
        MQ = np.sqrt((Qs.astype(np.float64) ** 2).sum(1)).max()
        MK = np.sqrt((Ks.astype(np.float64) ** 2).sum(1)).max()
        tol = 128 * 2.0 ** -24 * MQ * MK / math.sqrt(128) + 1e-9
        assert np.abs(dg - dev_ref).max() <= tol, (h, np.abs(dg - dev_ref).max(), tol)
        assert (dg <= Ug + tol).all()


def test_deviation_fullsize_C_properties(ba):
    """Full-size C (32 q-heads, 131072 tokens): U >= max_dev everywhere, the
    Pearson correlation of U and max_dev per head is informative (R > 0.5, the
    paper's criterion), and sampled block pairs equal the oracle's
    brute force on the same sorted rows."""
    w = CONFIGS["C"]
    q, k, v = make_qkv(w, device="cuda")
    ctx = ba.Context(q, k, v, 128, 0.5, diagnostics=True)
    sel = ctx.select(q, k, v)
    U, dev = ctx.deviation()
    torch.cuda.synchronize()
    assert torch.isfinite(U).all() and torch.isfinite(dev).all()
    MQ = sel.q_sorted.float().norm(dim=-1).amax(-1)  # [b, Hq]
    MK = sel.k_sorted.float().norm(dim=-1).amax(-1)
    tol = (128 * 2.0 ** -24 / math.sqrt(128)) * (MQ[0][:, None] * MK[0].repeat_interleave(4)[:, None]).double() + 1e-9
    assert (dev[0].flatten(1) <= U[0].flatten(1) + tol).all()
    x = U[0].flatten(1) - U[0].flatten(1).mean(-1, keepdim=True)
    y = dev[0].flatten(1) - dev[0].flatten(1).mean(-1, keepdim=True)
    r = (x * y).sum(-1) / (x.norm(dim=-1) * y.norm(dim=-1))
    assert (r > 0.5).all(), r
    rng = np.random.default_rng(5)
    for _ in range(6):
        h, gq, gk = int(rng.integers(32)), int(rng.integers(1024)), int(rng.integers(1024))
        Qb = sel.q_sorted[0, h, gq * 128:(gq + 1) * 128].double().cpu().numpy()
        Kb = sel.k_sorted[0, h // 4, gk * 128:(gk + 1) * 128].double().cpu().numpy()
        ref = O.max_logit_deviation(Qb, Kb, 128)[0, 0]
        assert abs(float(dev[0, h, gq, gk]) - ref) <= float(tol[h, 0]), (h, gq, gk)
