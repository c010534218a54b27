"""BA-Att CPU oracle — TEST INFRASTRUCTURE ONLY.

This module is the plain, slow, obviously-correct fp64 reference for the hot
path of Block Approximate Sparse Attention (arXiv 2605.19726).  It exists to
prove the CUDA path right.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  The
product package (``paper_2605_19726_b200``) never imports it and shares no code
with it; the only shared module is ``synth`` (seeded input generators, no
method arithmetic).

Citation key: ``P:n`` = line n of the paper text; section, equation
or algorithm label given beside it.  Readings of silent / garbled passages are
the ``A*`` items listed in DESIGN.md ("Readings of the paper").

Every value is float64 (inputs are upcast losslessly from the bf16 / fp32
values the GPU consumed).  Library primitives used as single steps: numpy
matmul, argsort(kind="stable"), exp, lexsort.  No blocking, fusion or
reordering beyond what the cited definition states.

Pin status (see tests/test_oracle_pins.py):
  norm_key, norm_rank, apply/unapply_permutation, make_grid, block_stats,
  block_logits, compensation_diag, compensation_exact, softmax_rows,
  kappa_from_density, topk_mask, topp_mask, select_head, block_sparse_attention_head,
  dense_attention, oracle_block_mass, deviation_bound, max_logit_deviation, lemma_check,
  ba_attention — all pinned (closed forms, worked examples, brute force,
  invariants).  Nothing here is "parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

SORT_NONE, SORT_Q, SORT_K, SORT_QK = 0, 1, 2, 3
COMP_NONE, COMP_DIAG, COMP_EXACT = 0, 1, 2


def _f64(x) -> np.ndarray:
    """Upcast any array-like (numpy / torch CPU tensor) to a float64 ndarray."""
    if hasattr(x, "detach"):  # torch tensor: go through float32 (exact for bf16/fp32)
        x = x.detach().to("cpu").float().numpy()
    return np.asarray(x, dtype=np.float64)


# --------------------------------------------------------------------------
# Softmax — P:249-250 (Eq. sdpa), P:289-291 (Eq. block-logit, m = softmax(l)).
# --------------------------------------------------------------------------
def softmax_rows(x) -> np.ndarray:
    """Row softmax exp(x_j) / sum_j' exp(x_j'), max-subtracted."""
    x = _f64(x)
    z = x - x.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


# --------------------------------------------------------------------------
# Norm-based ranking — P:436-446 (§3.3), Alg. 1 steps 1-2.
# --------------------------------------------------------------------------
def norm_key(X) -> np.ndarray:
    """Sort key of each row: ||x||_2^2 in fp32 with the fixed order of
    reading A4.

    P:438 defines the score s_j = ||K_j||_2; sorting by ||x||^2 gives the same
    order (monotone map).  The paper fixes no precision; reading A4 makes the
    key bit-defined in IEEE fp32 (round-to-nearest-even, no fused multiply-add):
    the d features are split into 16 contiguous parts of d/16; each part sums
    x*x sequentially (product rounded, then sum rounded); the 16 partial sums
    are combined by the halving tree p[:8]+p[8:], then [:4]+[4:], [:2]+[2:],
    [0]+[1].  d not divisible by 16 is zero-padded.  (The key only ranks rows;
    its fp32 rounding error, <= 13 u relative, changes nothing but the order of
    near-equal norms, and both sides round identically.)
    """
    X = _f64(X).astype(np.float32)  # exact: inputs are bf16 / fp32 values
    L, d = X.shape
    if d % 16:  # zero features add exactly 0: pad to a multiple of 16
        X = np.concatenate([X, np.zeros((L, 16 - d % 16), dtype=np.float32)], axis=1)
        d = X.shape[1]
    parts = X.reshape(L, 16, d // 16)
    p = np.zeros((L, 16), dtype=np.float32)
    for t in range(d // 16):  # sequential within each part, fp32 ops
        sq = parts[:, :, t] * parts[:, :, t]
        p = p + sq
    a = p[:, :8] + p[:, 8:]
    a = a[:, :4] + a[:, 4:]
    a = a[:, :2] + a[:, 2:]
    a = a[:, 0] + a[:, 1]
    return a.astype(np.float32)


def norm_rank(X, window: Optional[int] = None) -> np.ndarray:
    """pi with s_pi(1) <= s_pi(2) <= ...; pi maps sorted position
    -> original index.  Ties -> lower original index (stable sort, reading A3).
    ``window``: Alg. 1's "(windowed) sort" — every run of ``window``
    consecutive tokens is sorted independently (reading A5; default global)."""
    key = norm_key(X)
    L = key.shape[0]
    if window is None or window <= 0 or window >= L:
        return np.argsort(key, kind="stable").astype(np.int64)
    out = np.empty(L, dtype=np.int64)
    for s in range(0, L, window):
        e = min(s + window, L)
        out[s:e] = s + np.argsort(key[s:e], kind="stable")
    return out


def apply_permutation(X, perm) -> np.ndarray:
    """X'_i = X_{pi(i)}."""
    return _f64(X)[np.asarray(perm)]


def unapply_permutation(Xs, perm) -> np.ndarray:
    """O[pi(i)] = O'_i — remap to the original order via pi^{-1}."""
    Xs = _f64(Xs)
    out = np.empty_like(Xs)
    out[np.asarray(perm)] = Xs
    return out


# --------------------------------------------------------------------------
# Block partition and statistics — P:260, Alg. 1 steps 3-4,
# P:516 (first/second moments).
# --------------------------------------------------------------------------
def make_grid(L: int, B: int) -> list[tuple[int, int]]:
    """I(g) = [gB, min((g+1)B, L)), N = ceil(L/B); ragged last block allowed
    (P:260 assumes B | L; reading A11)."""
    assert L >= 1 and B >= 1
    return [(s, min(s + B, L)) for s in range(0, L, B)]


def block_stats(X, B: int):
    """Per block g: mean Xbar_g ("mean pooling"), per-dimension
    population variance Var[X_t]_g = (1/n_g) sum (x_t - Xbar_t)^2 (P:516,
    reading A8; two-pass), and the count n_g.  Returns (mean[N,d], var[N,d],
    count[N])."""
    X = _f64(X)
    grid = make_grid(X.shape[0], B)
    mean = np.stack([X[s:e].mean(axis=0) for s, e in grid])
    var = np.stack([((X[s:e] - mean[g]) ** 2).mean(axis=0) for g, (s, e) in enumerate(grid)])
    count = np.array([e - s for s, e in grid], dtype=np.int64)
    return mean, var, count


def block_covariance(X, B: int) -> np.ndarray:
    """Full population covariance Sigma_g = E_i[dX_i dX_i^T].
    Diagnostic / NEXT-4 only (O(L d^2))."""
    X = _f64(X)
    out = []
    for s, e in make_grid(X.shape[0], B):
        D = X[s:e] - X[s:e].mean(axis=0)
        out.append(D.T @ D / (e - s))
    return np.stack(out)


# --------------------------------------------------------------------------
# Block logits and compensation — Eq. block-logit,
# Eq. cov-comp, Eq. diag-variance-form,
# Alg. 1 steps 5-7.
# --------------------------------------------------------------------------
def block_logits(q_mean, k_mean, d: int) -> np.ndarray:
    """l_{gq,gk} = (Qbar_gq . Kbar_gk) / sqrt(d)."""
    return _f64(q_mean) @ _f64(k_mean).T / math.sqrt(d)


def compensation_diag(q_mean, q_var, k_mean, k_var, d: int) -> np.ndarray:
    """Delta = (1/d) sum_t ( Var[Q_t] Kbar_t^2 + Var[K_t] Qbar_t^2
                            + Var[Q_t] Var[K_t] )."""
    qm, qv, km, kv = _f64(q_mean), _f64(q_var), _f64(k_mean), _f64(k_var)
    return (qv @ (km * km).T + (qm * qm) @ kv.T + qv @ kv.T) / d


def compensation_exact(q_cov, k_cov, d: int) -> np.ndarray:
    """Delta = (1/d) tr(Sigma^Q_gq Sigma^K_gk).  NEXT-4."""
    qc, kc = _f64(q_cov), _f64(k_cov)
    # tr(A B) = sum_{s,t} A[s,t] B[t,s]
    return np.einsum("ast,bts->ab", qc, kc) / d


def kappa_from_density(density: float, n_k: int) -> int:
    """Per-query-block budget kappa (Alg. 1 REQUIRE; step 10).
    Reading A2: kappa = max(1, min(N_k, floor(density * N_k + 1/2))) in fp64."""
    assert 0.0 < density <= 1.0
    return max(1, min(n_k, int(math.floor(float(density) * n_k + 0.5))))


def topk_mask(m, kappa: int):
    """Alg. 1 step 10: per row select the top-kappa key blocks by
    m'; ties -> lower g_k (reading A3).  Returns (mask[Nq,Nk] uint8,
    tau[Nq] = m' of the kappa-th selected entry, kv_index[Nq,kappa] ascending).
    """
    m = _f64(m)
    nq, nk = m.shape
    mask = np.zeros((nq, nk), dtype=np.uint8)
    tau = np.zeros(nq, dtype=np.float64)
    idx = np.zeros((nq, kappa), dtype=np.int64)
    cols = np.arange(nk)
    for r in range(nq):
        order = np.lexsort((cols, -m[r]))  # primary: -m' (desc), secondary: g_k (asc)
        chosen = order[:kappa]
        mask[r, chosen] = 1
        tau[r] = m[r, order[kappa - 1]]
        idx[r] = np.sort(chosen)
    return mask, tau, idx


def topp_mask(m, top_p: float, kappa_cap: int):
    """Cumulative-mass budget (NEXT-1; the paper builds M from m' "under
    different computational budgets").  Reading A23: per row, order the
    key blocks by (-m', g_k) as in top-kappa (reading A3) and keep the shortest
    prefix whose cumulative mass reaches top_p:
        kappa_row = min{k >= 1 : sum_{r<k} m'_(r) >= top_p}   (N_k if none),
    then cap it at kappa_cap (the density budget; density 1 = no cap).  The
    cumulative sum runs sequentially in that order, in fp64.  Returns (mask,
    tau = m' of the last kept entry, kv_index as a list of ascending arrays,
    kappa_row[Nq])."""
    m = _f64(m)
    nq, nk = m.shape
    assert 0.0 < top_p <= 1.0 and 1 <= kappa_cap <= nk
    mask = np.zeros((nq, nk), dtype=np.uint8)
    tau = np.zeros(nq, dtype=np.float64)
    kap = np.zeros(nq, dtype=np.int64)
    idx = []
    cols = np.arange(nk)
    for r in range(nq):
        order = np.lexsort((cols, -m[r]))
        cum = np.cumsum(m[r, order])
        hit = np.nonzero(cum >= top_p)[0]
        k = int(hit[0]) + 1 if hit.size else nk
        k = min(k, kappa_cap)
        chosen = order[:k]
        mask[r, chosen] = 1
        tau[r] = m[r, order[k - 1]]
        kap[r] = k
        idx.append(np.sort(chosen))
    return mask, tau, idx, kap


@dataclass
class Selection:
    perm_q: np.ndarray
    perm_k: np.ndarray
    q_mean: np.ndarray
    q_var: np.ndarray
    k_mean: np.ndarray
    k_var: np.ndarray
    logits: np.ndarray       # l
    delta: np.ndarray        # Delta
    lprime: np.ndarray       # l' = l + beta Delta
    m: np.ndarray            # m' = softmax_row(l')
    mask: np.ndarray
    tau: np.ndarray
    kv_index: np.ndarray
    kappa: int
    extra: dict = field(default_factory=dict)


def select_head(Q, K, B: int, density: float, beta: float = 1.0,
                sort: int = SORT_QK, comp: int = COMP_DIAG,
                window: Optional[int] = None,
                perm_q=None, perm_k=None, top_p: Optional[float] = None) -> Selection:
    """Algorithm 1 steps 1-10 for one (batch, q-head) with its
    key head.  ``perm_q``/``perm_k`` may be supplied (e.g. shared K-side
    permutation under GQA) — otherwise computed here.  ``top_p``: the
    cumulative-mass budget (reading A23) instead of top-kappa, capped at the
    density's kappa; ``kv_index`` is then a list of per-row arrays."""
    Q, K = _f64(Q), _f64(K)
    d = Q.shape[1]
    if perm_q is None:  # step 1
        perm_q = norm_rank(Q, window) if sort in (SORT_Q, SORT_QK) else np.arange(Q.shape[0])
    if perm_k is None:  # step 2
        perm_k = norm_rank(K, window) if sort in (SORT_K, SORT_QK) else np.arange(K.shape[0])
    Qs, Ks = apply_permutation(Q, perm_q), apply_permutation(K, perm_k)
    q_mean, q_var, _ = block_stats(Qs, B)          # steps 3-4
    k_mean, k_var, _ = block_stats(Ks, B)
    l = block_logits(q_mean, k_mean, d)             # step 5
    if comp == COMP_DIAG:                           # step 6
        delta = compensation_diag(q_mean, q_var, k_mean, k_var, d)
    elif comp == COMP_EXACT:
        delta = compensation_exact(block_covariance(Qs, B), block_covariance(Ks, B), d)
    else:
        delta = np.zeros_like(l)
    lp = l + float(beta) * delta                    # step 7
    m = softmax_rows(lp)                            # step 9
    kappa = kappa_from_density(density, l.shape[1])
    extra = {}
    if top_p is None:
        mask, tau, idx = topk_mask(m, kappa)        # step 10
    else:
        mask, tau, idx, extra["kappa_row"] = topp_mask(m, top_p, kappa)
        extra["top_p"] = float(top_p)
    return Selection(np.asarray(perm_q), np.asarray(perm_k), q_mean, q_var, k_mean, k_var,
                     l, delta, lp, m, mask, tau, idx, kappa, extra)


# --------------------------------------------------------------------------
# Attention — Eq. sdpa; block-sparse execution (P:263-264,
# Alg. 1 steps 11-12).
# --------------------------------------------------------------------------
def block_sparse_attention_head(Qs, Ks, Vs, kv_index, B: int, scale: float,
                                q_blocks: Optional[Sequence[int]] = None):
    """For every query i in I(g_q): softmax over the keys j of the selected
    blocks only, renormalised over that support (reading A16),
    O'_i = sum_j P_ij V'_j.  Inputs are the *sorted* Q', K', V'.  Returns
    (O' [Lq, dv], lse [Lq]) in sorted order; rows of unrequested q-blocks are
    NaN.  ``kv_index[g_q]`` lists the selected g_k."""
    Qs, Ks, Vs = _f64(Qs), _f64(Ks), _f64(Vs)
    gq_grid = make_grid(Qs.shape[0], B)
    gk_grid = make_grid(Ks.shape[0], B)
    out = np.full((Qs.shape[0], Vs.shape[1]), np.nan)
    lse = np.full(Qs.shape[0], np.nan)
    blocks = range(len(gq_grid)) if q_blocks is None else q_blocks
    for g in blocks:
        s, e = gq_grid[g]
        cols = np.concatenate([np.arange(*gk_grid[int(j)]) for j in kv_index[g]])
        S = Qs[s:e] @ Ks[cols].T * scale
        mx = S.max(axis=1, keepdims=True)
        P = np.exp(S - mx)
        den = P.sum(axis=1, keepdims=True)
        out[s:e] = (P / den) @ Vs[cols]
        lse[s:e] = (mx + np.log(den))[:, 0]
    return out, lse


def dense_attention(Q, K, V, scale: Optional[float] = None, row_block: int = 1024):
    """O = softmax(Q K^T / sqrt(d)) V, computed one row block at a
    time so the L x L map is never held whole."""
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    if scale is None:
        scale = 1.0 / math.sqrt(Q.shape[1])
    out = np.empty((Q.shape[0], V.shape[1]))
    for s in range(0, Q.shape[0], row_block):
        S = Q[s:s + row_block] @ K.T * scale
        out[s:s + row_block] = softmax_rows(S) @ V
    return out


def dense_attention_map(Q, K, scale: Optional[float] = None) -> np.ndarray:
    """A = softmax(Q K^T / sqrt(d)), materialised (small L only)."""
    Q, K = _f64(Q), _f64(K)
    if scale is None:
        scale = 1.0 / math.sqrt(Q.shape[1])
    return softmax_rows(Q @ K.T * scale)


def oracle_block_mass(A, Bq: int, Bk: int) -> np.ndarray:
    """m_hat_{gq,gk} = (1/|I(gq)|) sum_{i in I(gq)} sum_{j in J(gk)} A_ij
    (Eq. oracle-dist)."""
    A = _f64(A)
    gq, gk = make_grid(A.shape[0], Bq), make_grid(A.shape[1], Bk)
    out = np.empty((len(gq), len(gk)))
    for a, (s, e) in enumerate(gq):
        for b, (u, v) in enumerate(gk):
            out[a, b] = A[s:e, u:v].sum() / (e - s)
    return out


# --------------------------------------------------------------------------
# Diagnostics — Eq. logits-bound, Lemma 1.
# --------------------------------------------------------------------------
def deviation_bound(Xq, Xk, B: int):
    """U = (R^Q M^K + M^Q R^K + R^Q R^K) / sqrt(d) per block pair, with
    R = max ||x - xbar||, M = max ||x|| over the block."""
    Xq, Xk = _f64(Xq), _f64(Xk)
    d = Xq.shape[1]

    def rm(X):
        R, M = [], []
        for s, e in make_grid(X.shape[0], B):
            mu = X[s:e].mean(axis=0)
            R.append(np.sqrt(((X[s:e] - mu) ** 2).sum(axis=1)).max())
            M.append(np.sqrt((X[s:e] ** 2).sum(axis=1)).max())
        return np.array(R), np.array(M)

    RQ, MQ = rm(Xq)
    RK, MK = rm(Xk)
    return (np.outer(RQ, MK) + np.outer(MQ, RK) + np.outer(RQ, RK)) / math.sqrt(d)


def max_logit_deviation(Xq, Xk, B: int):
    """max_{i in I(g_q), j in J(g_k)} |l_hat_ij - l_{g_q,g_k}| per block pair, with
    l_hat_ij = Q_i . K_j / sqrt(d) (the token logit) and l = Qbar . Kbar / sqrt(d)
    (Eq. block-logit): the "observed maximum logit deviation" that Fig. 2
     plots against U (Eq. logit-deviation).  Brute force over
    every token pair of every block pair."""
    Xq, Xk = _f64(Xq), _f64(Xk)
    d = Xq.shape[1]
    gq, gk = make_grid(Xq.shape[0], B), make_grid(Xk.shape[0], B)
    out = np.empty((len(gq), len(gk)))
    for a, (s, e) in enumerate(gq):
        qbar = Xq[s:e].mean(axis=0)
        for b, (u, v) in enumerate(gk):
            kbar = Xk[u:v].mean(axis=0)
            tok = Xq[s:e] @ Xk[u:v].T / math.sqrt(d)
            out[a, b] = np.abs(tok - (qbar @ kbar) / math.sqrt(d)).max()
    return out


def lemma_check(u, v):
    """Lemma 1 (proof P:38-90): returns (lhs, 2 min(1/a,1/b)||u-v||_1,
    4/(a+b) ||u-v||_1) for positive u, v."""
    u, v = _f64(u), _f64(v)
    assert (u > 0).all() and (v > 0).all()
    a, b = u.sum(), v.sum()
    d1 = np.abs(u - v).sum()
    lhs = np.abs(u / a - v / b).sum()
    return lhs, 2.0 * min(1.0 / a, 1.0 / b) * d1, 4.0 / (a + b) * d1


# --------------------------------------------------------------------------
# Whole path, multi-head — Alg. 1 per (batch, q-head); GQA
# reading A14 (perm_k, K', V', K-stats per KV head).
# --------------------------------------------------------------------------
@dataclass
class Params:
    block_size: int = 128
    density: float = 0.5
    beta: float = 1.0
    sort: int = SORT_QK
    comp: int = COMP_DIAG
    window: Optional[int] = None
    scale: Optional[float] = None
    top_p: Optional[float] = None   # cumulative-mass budget (reading A23); None = top-kappa


def ba_attention(Q, K, V, p: Params, q_blocks: Optional[dict] = None,
                 selections: Optional[dict] = None):
    """Q [b,Hq,Lq,d], K,V [b,Hkv,Lk,d] (any float array-like) -> O [b,Hq,Lq,dv]
    in the ORIGINAL token order, plus the per-head Selection objects.

    ``q_blocks``: optional {(b,hq): [g_q,...]} to evaluate only some query
    blocks (sampled parity at full size); other rows are NaN.
    ``selections``: optional {(b,hq): (perm_q, perm_k, kv_index)} to run the
    attention half with a given selection (reading A16: output parity uses
    the GPU's mask and permutations after those are checked)."""
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    b, hq, lq, d = Q.shape
    hkv = K.shape[1]
    assert hq % hkv == 0
    grp = hq // hkv
    scale = p.scale if p.scale else 1.0 / math.sqrt(d)
    O = np.full((b, hq, lq, V.shape[3]), np.nan)
    sels = {}
    for bi in range(b):
        kperm_cache = {}
        for h in range(hq):
            hk = h // grp
            if selections is not None:
                perm_q, perm_k, kv_index = selections[(bi, h)]
                perm_q, perm_k = np.asarray(perm_q), np.asarray(perm_k)
                kv_index = [np.asarray(r) for r in kv_index]
            else:
                if hk not in kperm_cache:
                    kperm_cache[hk] = (norm_rank(K[bi, hk], p.window) if p.sort in (SORT_K, SORT_QK)
                                       else np.arange(K.shape[2]))
                sel = select_head(Q[bi, h], K[bi, hk], p.block_size, p.density, p.beta,
                                  p.sort, p.comp, p.window, perm_k=kperm_cache[hk], top_p=p.top_p)
                sels[(bi, h)] = sel
                perm_q, perm_k, kv_index = sel.perm_q, sel.perm_k, sel.kv_index
            Qs = apply_permutation(Q[bi, h], perm_q)
            Ks = apply_permutation(K[bi, hk], perm_k)
            Vs = apply_permutation(V[bi, hk], perm_k)
            qb = None if q_blocks is None else q_blocks.get((bi, h), [])
            Os, _ = block_sparse_attention_head(Qs, Ks, Vs, kv_index, p.block_size, scale, qb)
            O[bi, h] = unapply_permutation(Os, perm_q)
    return O, sels


def sparse_flops(kv_index, Lq: int, Lk: int, B: int, d: int, dv: Optional[int] = None) -> int:
    """Algorithmic FLOPs of the selected pairs: sum over M of
    2 n_q n_k d (QK^T) + 2 n_q n_k dv (PV), actual ragged sizes."""
    dv = d if dv is None else dv
    gq, gk = make_grid(Lq, B), make_grid(Lk, B)
    tot = 0
    for g, row in enumerate(kv_index):
        nq = gq[g][1] - gq[g][0]
        for j in row:
            nk = gk[int(j)][1] - gk[int(j)][0]
            tot += 2 * nq * nk * (d + dv)
    return tot
