"""Parity helpers: compare the CUDA path (through the C ABI) with the oracle.

Contract:
  P1 perm_q / perm_k exact;  P2 block stats (diagnostic);  P3 m' (diagnostic);
  P4 masks equal except entries with |m'_ref - tau_ref| <= 1e-6, kv_count =
  kappa, lists ascending;  P5 outputs within 2e-2 (bf16) / 1e-5 (fp32) of the
  oracle run with the GPU's permutations and mask (reading A16);  P6 rho = 1
  equals dense.
"""
from __future__ import annotations

import math

import numpy as np
import torch

import oracle as O

MASK_BAND = 1e-6
TOL = {torch.bfloat16: 2e-2, torch.float32: 1e-5}
SORT_CODE = {"none": O.SORT_NONE, "q": O.SORT_Q, "k": O.SORT_K, "qk": O.SORT_QK}
COMP_CODE = {"none": O.COMP_NONE, "diag": O.COMP_DIAG, "exact": O.COMP_EXACT}


def oracle_select_all(q, k, B, density, beta, sort, comp, window=None, heads=None, top_p=None):
    """Oracle selection for every (b, hq) (or the listed heads) on the exact
    tensors the GPU consumed."""
    b, hq = q.shape[0], q.shape[1]
    grp = hq // k.shape[1]
    qn = q.detach().cpu().float().numpy()
    kn = k.detach().cpu().float().numpy()
    out = {}
    kcache = {}
    for bi in range(b):
        for h in (range(hq) if heads is None else heads):
            hk = h // grp
            if (bi, hk) not in kcache:
                kcache[(bi, hk)] = (O.norm_rank(kn[bi, hk], window) if SORT_CODE[sort] in (O.SORT_K, O.SORT_QK)
                                    else np.arange(kn.shape[2]))
            out[(bi, h)] = O.select_head(qn[bi, h], kn[bi, hk], B, density, beta, SORT_CODE[sort],
                                         COMP_CODE[comp], window, perm_k=kcache[(bi, hk)], top_p=top_p)
    return out


def check_selection(sel, ref: dict, band: float = MASK_BAND, check_stats: bool = True):
    """P1-P4.  Returns a report dict; raises AssertionError on a gate failure."""
    rep = {"perm_mismatch": 0, "mask_mismatch": 0, "mask_in_band": 0, "band_population": 0,
           "max_abs_dm": 0.0, "max_abs_dm_near_tau": 0.0, "max_stat_err": 0.0}
    perm_q = sel.perm_q.cpu().numpy()
    perm_k = sel.perm_k.cpu().numpy()
    kv_index = sel.kv_index.cpu().numpy()
    kv_count = sel.kv_count.cpu().numpy()
    mask = sel.mask.cpu().numpy() if sel.mask is not None else None
    prob = sel.block_prob.cpu().numpy() if sel.block_prob is not None else None
    hq = perm_q.shape[1]
    grp = hq // perm_k.shape[1]
    for (bi, h), r in ref.items():
        hk = h // grp
        rep["perm_mismatch"] += int((perm_q[bi, h] != r.perm_q).sum()) + int((perm_k[bi, hk] != r.perm_k).sum())
        gmask = np.zeros_like(r.mask)
        if "kappa_row" not in r.extra:  # top-kappa: every row keeps exactly kappa
            assert (kv_count[bi, h] == r.kappa).all(), "kv_count != kappa"
            idx = kv_index[bi, h]
            assert (np.diff(idx, axis=1) > 0).all(), "kv_index rows must be strictly ascending"
            np.put_along_axis(gmask, idx.astype(np.int64), 1, axis=1)
            near = np.abs(r.m - r.tau[:, None]) <= band
        else:  # top-p (reading A23): kappa_row may differ only where the cumulative mass ties p
            kr = r.extra["kappa_row"]
            near = np.abs(r.m - r.tau[:, None]) <= band
            for g in range(kr.shape[0]):
                c = int(kv_count[bi, h, g])
                row = kv_index[bi, h, g, :c]
                assert c >= 1 and (np.diff(row) > 0).all(), "kv_index rows must be strictly ascending"
                gmask[g, row] = 1
                if c != kr[g]:
                    # the prefix masses between the two lengths all lie within the band of p
                    order = np.lexsort((np.arange(r.m.shape[1]), -r.m[g]))
                    cum = np.cumsum(r.m[g, order])
                    lo, hi = min(c, int(kr[g])), max(c, int(kr[g]))
                    assert np.abs(cum[lo - 1:hi - 1] - r.extra["top_p"]).max() <= band, \
                        f"P4 kappa_row {c} != {kr[g]} away from the cumulative-mass boundary"
                    rep["kappa_row_in_band"] = rep.get("kappa_row_in_band", 0) + 1
                    near[g, order[lo:hi]] = True
        if mask is not None:
            assert (mask[bi, h] == gmask).all(), "mask and kv_index disagree"
        diff = gmask != r.mask
        rep["band_population"] += int(near.sum())
        rep["mask_mismatch"] += int((diff & ~near).sum())
        rep["mask_in_band"] += int((diff & near).sum())
        if prob is not None:
            dm = np.abs(prob[bi, h] - r.m)
            rep["max_abs_dm"] = max(rep["max_abs_dm"], float(dm.max()))
            n2 = np.abs(r.m - r.tau[:, None]) <= 1e-4
            if n2.any():
                rep["max_abs_dm_near_tau"] = max(rep["max_abs_dm_near_tau"], float(dm[n2].max()))
        if check_stats and sel.q_mean is not None:
            for g_t, r_t in ((sel.q_mean[bi, h], r.q_mean), (sel.q_var[bi, h], r.q_var),
                             (sel.k_mean[bi, hk], r.k_mean), (sel.k_var[bi, hk], r.k_var)):
                e = np.abs(g_t.cpu().numpy() - r_t) / (1 + np.abs(r_t))
                rep["max_stat_err"] = max(rep["max_stat_err"], float(e.max()))
    assert rep["perm_mismatch"] == 0, f"P1 permutation mismatch: {rep}"
    assert rep["mask_mismatch"] == 0, f"P4 mask mismatch outside the band: {rep}"
    return rep


def oracle_output_with_gpu_selection(q, k, v, sel, B, scale=None, q_blocks=None):
    """O10-O11 on the GPU's permutations and kv_index (reading A16)."""
    b, hq = q.shape[0], q.shape[1]
    selections = {}
    pq, pk, idx = sel.perm_q.cpu().numpy(), sel.perm_k.cpu().numpy(), sel.kv_index.cpu().numpy()
    cnt = sel.kv_count.cpu().numpy()
    grp = hq // k.shape[1]
    for bi in range(b):
        for h in range(hq):
            rows = [idx[bi, h, g, :cnt[bi, h, g]] for g in range(idx.shape[2])]
            selections[(bi, h)] = (pq[bi, h], pk[bi, h // grp], rows)
    p = O.Params(block_size=B, scale=scale)
    out, _ = O.ba_attention(q, k, v, p, q_blocks=q_blocks, selections=selections)
    return out


def max_abs_err(gpu: torch.Tensor, ref: np.ndarray) -> float:
    g = gpu.detach().cpu().double().numpy()
    m = ~np.isnan(ref)
    return float(np.abs(g[m] - ref[m]).max()) if m.any() else 0.0
