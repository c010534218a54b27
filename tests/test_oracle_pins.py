"""Pins for the CPU oracle (runs with -m "not gpu").

Each test pins an oracle function to something other than itself: a worked
example printed in the paper/SPEC (tests/golden/worked_examples.json, cited
there), a closed form, a theorem, an invariant, or brute force on tiny
inputs.  Chosen so that a dropped term, a wrong sign / index or a transposed
operand in oracle/ba_oracle.py fails at least one of them.
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle as O
from synth import CONFIGS, constant_block_qkv, make_qkv

RNG = np.random.default_rng(20260519)


# ---------------------------------------------------------------- softmax
@pytest.mark.parametrize("key", ["softmax_123", "softmax_uniform", "softmax_ln2"])
def test_softmax_worked(golden, key):
    g = golden[key]
    np.testing.assert_allclose(O.softmax_rows(np.array([g["x"]]))[0], g["expected"], atol=g["tol"], rtol=0)


def test_softmax_shift_invariance_and_sum():
    x = RNG.uniform(-50, 50, size=(64, 33))
    a, b = O.softmax_rows(x), O.softmax_rows(x + 17.25)
    np.testing.assert_allclose(a, b, atol=1e-12, rtol=0)
    np.testing.assert_allclose(a.sum(axis=1), 1.0, atol=1e-12)
    assert (a.argmax(1) == x.argmax(1)).all()


# ---------------------------------------------------------------- Lemma 1
def test_lemma_worked(golden):
    g = golden["lemma_example"]
    lhs, tight, final = O.lemma_check(g["u"], g["v"])
    assert lhs == pytest.approx(g["lhs"], abs=1e-15)
    assert tight == pytest.approx(g["tight"], abs=1e-15)
    assert final == pytest.approx(g["final"], abs=1e-15)


def test_lemma_chain_random():
    """||pi(u)-pi(v)||_1 <= 2 min(1/a,1/b)||u-v||_1 <= 4/(a+b)||u-v||_1
    on 1e5 random positive pairs."""
    n = 100_000
    lens = RNG.integers(2, 65, size=n)
    worst = -np.inf
    for L in np.unique(lens):
        k = int((lens == L).sum())
        u = RNG.uniform(1e-6, 100, size=(k, L))
        v = RNG.uniform(1e-6, 100, size=(k, L))
        a, b = u.sum(1), v.sum(1)
        d1 = np.abs(u - v).sum(1)
        lhs = np.abs(u / a[:, None] - v / b[:, None]).sum(1)
        tight = 2 * np.minimum(1 / a, 1 / b) * d1
        final = 4 / (a + b) * d1
        worst = max(worst, float((lhs - tight).max()), float((tight - final).max()))
    assert worst <= 1e-12
    # the oracle's lemma_check agrees with the vectorised statement on a sample
    u, v = RNG.uniform(1e-3, 100, 9), RNG.uniform(1e-3, 100, 9)
    lhs, tight, final = O.lemma_check(u, v)
    assert lhs <= tight + 1e-12 and tight <= final + 1e-12


def test_softmax_as_normalisation_lemma():
    """softmax(l) = pi(exp(l)); Lemma 1 bounds the block-distribution change
    by the change of exp-logits."""
    l1 = RNG.normal(size=20)
    l2 = l1 + RNG.normal(scale=1e-2, size=20)
    gap = np.abs(O.softmax_rows(l1[None])[0] - O.softmax_rows(l2[None])[0]).sum()
    lhs, tight, final = O.lemma_check(np.exp(l1), np.exp(l2))
    assert gap == pytest.approx(lhs, abs=1e-14)
    assert gap <= final + 1e-12


# ---------------------------------------------------------------- norms and ranking
@pytest.mark.parametrize("key", ["norm_34", "norm_1111"])
def test_norm_key_worked(golden, key):
    g = golden[key]
    row = np.zeros((1, 16), dtype=np.float64)
    row[0, :len(g["row"])] = g["row"]
    assert float(O.norm_key(row)[0]) == g["expected_norm"] ** 2


def test_norm_key_error_bound():
    """The A4 key is the fp32 sum of squares: within the recursive-summation
    bound (d/16 sequential adds + 4 tree levels + the product rounding, all
    with unit roundoff u = 2^-24) of the exact rational ||x||^2, for bf16 and
    fp32 rows of heavy-tailed magnitude.  A dropped, doubled or mis-squared
    term breaks it by far more than the bound."""
    for dt in (torch.bfloat16, torch.float32):
        x = (torch.randn(200, 128) * torch.exp(torch.randn(200, 1) * 2)).to(dt).float().numpy().astype(np.float64)
        keys = O.norm_key(x)
        n_ops = 128 // 16 + 4 + 1
        for r in range(x.shape[0]):
            exact = sum(Fraction(float(v)) ** 2 for v in x[r])
            err = abs(Fraction(float(keys[r])) - exact)
            assert err <= Fraction(n_ops, 1 << 24) * exact * Fraction(101, 100)
    # small integers: every partial sum is exact in fp32 -> the exact value
    x = RNG.integers(-50, 50, size=(20, 64)).astype(np.float64)
    np.testing.assert_array_equal(O.norm_key(x), (x * x).sum(1).astype(np.float32))


def test_norm_key_order_is_the_definition():
    """fp32 sums depend on the order, so the oracle must follow the stated
    tree: check it against a scalar re-statement of A4 with np.float32 scalar
    arithmetic on random fp32 rows of wide dynamic range."""
    x = (RNG.standard_normal((50, 64)) * np.exp(RNG.normal(size=(50, 64)) * 3)).astype(np.float32)
    keys = O.norm_key(x.astype(np.float64))
    for r in range(50):
        p = []
        for lane in range(16):
            s = np.float32(0.0)
            for t in range(4):
                v = x[r, lane * 4 + t]
                s = np.float32(s + np.float32(v * v))
            p.append(s)
        while len(p) > 1:
            h = len(p) // 2
            p = [np.float32(p[i] + p[i + h]) for i in range(h)]
        assert p[0] == keys[r]


def test_rank_worked(golden):
    g = golden["rank_312"]
    X = np.zeros((3, 16))
    X[:, 0] = g["norms"]
    assert list(O.norm_rank(X)) == g["expected_perm"]
    g = golden["rank_window"]
    X = np.zeros((4, 16))
    X[:, 0] = g["norms"]
    assert list(O.norm_rank(X, window=g["window"])) == g["expected_perm"]


def test_rank_invariants():
    X = RNG.standard_normal((500, 32))
    X[10] = X[3]  # exact tie
    X[400] = X[3]
    p = O.norm_rank(X)
    keys = O.norm_key(X)
    assert sorted(p.tolist()) == list(range(500))
    assert (np.diff(keys[p]) >= 0).all()
    # ties keep original order
    pos = {int(v): i for i, v in enumerate(p)}
    assert pos[3] < pos[10] < pos[400]
    # all-equal norms -> identity
    E = np.ones((37, 16))
    assert (O.norm_rank(E) == np.arange(37)).all()


def test_permutation_roundtrip():
    X = RNG.standard_normal((99, 8))
    p = RNG.permutation(99)
    assert (O.unapply_permutation(O.apply_permutation(X, p), p) == X).all()
    Xs = O.apply_permutation(X, p)
    assert (Xs[5] == X[p[5]]).all()


# ---------------------------------------------------------------- grid and stats
@pytest.mark.parametrize("key", ["grid_6_2", "grid_5_2", "grid_4_8"])
def test_grid_worked(golden, key):
    g = golden[key]
    assert [list(t) for t in O.make_grid(g["L"], g["B"])] == g["expected"]


@pytest.mark.parametrize("key", ["stats_sym_pair", "stats_three"])
def test_stats_worked(golden, key):
    g = golden[key]
    blk = np.array(g["block"])
    mean, var, cnt = O.block_stats(blk, blk.shape[0])
    np.testing.assert_allclose(mean[0], g["mean"], atol=1e-15)
    np.testing.assert_allclose(var[0], g["var"], atol=1e-15)
    assert cnt[0] == blk.shape[0]


def test_stats_ragged_and_constant():
    X = RNG.standard_normal((10, 4))
    X[4:8] = X[4]
    mean, var, cnt = O.block_stats(X, 4)
    assert list(cnt) == [4, 4, 2]
    np.testing.assert_allclose(mean[2], X[8:10].mean(0), atol=1e-15)
    assert (var[1] == 0).all()
    # brute force population variance
    for g, (s, e) in enumerate(O.make_grid(10, 4)):
        for t in range(4):
            vals = X[s:e, t]
            mu = sum(vals) / len(vals)
            bf = sum((v - mu) ** 2 for v in vals) / len(vals)
            assert var[g, t] == pytest.approx(bf, abs=1e-14)
    cov = O.block_covariance(X, 4)
    np.testing.assert_allclose(np.diagonal(cov, axis1=1, axis2=2), var, atol=1e-14)


# ---------------------------------------------------------------- logits and compensation
@pytest.mark.parametrize("key", ["logit_orth", "logit_sqrt2"])
def test_logits_worked(golden, key):
    g = golden[key]
    l = O.block_logits(np.array([g["qbar"]]), np.array([g["kbar"]]), g["d"])
    assert l[0, 0] == pytest.approx(g["expected"], abs=1e-15)


def test_logits_mean_of_token_logits():
    """mean_{(i,j) in IxJ} lhat_ij = l_{gq,gk} exactly (bilinearity; P:287,
    P:333) — also fixes the 1/sqrt(d) (not 1/d) scale and the operand order."""
    Q, K = RNG.standard_normal((24, 8)), RNG.standard_normal((40, 8))
    qm, _, _ = O.block_stats(Q, 8)
    km, _, _ = O.block_stats(K, 8)
    l = O.block_logits(qm, km, 8)
    tok = Q @ K.T / math.sqrt(8)
    for a, (s, e) in enumerate(O.make_grid(24, 8)):
        for b, (u, v) in enumerate(O.make_grid(40, 8)):
            assert l[a, b] == pytest.approx(tok[s:e, u:v].mean(), abs=1e-12)


def test_comp_worked(golden):
    g = golden["comp_29"]
    D = O.compensation_diag(np.array([g["qbar"]]), np.array([g["qvar"]]),
                            np.array([g["kbar"]]), np.array([g["kvar"]]), g["d"])
    assert D[0, 0] == g["expected"]


def _diag_cov_block(mean, sig):
    """2d tokens mean ± sig_t*sqrt(d) e_t: population covariance diag(sig^2)."""
    d = mean.shape[0]
    rows = []
    for t in range(d):
        e = np.zeros(d)
        e[t] = sig[t] * math.sqrt(d)
        rows += [mean + e, mean - e]
    return np.array(rows)


def test_comp_diag_equals_logit_variance_for_diagonal_cov():
    """Derived identity (SURVEY §0 finding 3): Var_{(i,j)}[lhat_ij] =
    (tr(SQ SK) + Qbar^T SK Qbar + Kbar^T SQ Kbar)/d; for diagonal covariances
    that is exactly Eq. diag-variance-form.  Brute force over all
    token pairs."""
    d = 4
    for _ in range(20):
        qb = _diag_cov_block(RNG.standard_normal(d), RNG.uniform(0.1, 2, d))
        kb = _diag_cov_block(RNG.standard_normal(d), RNG.uniform(0.1, 2, d))
        B = 2 * d
        qm, qv, _ = O.block_stats(qb, B)
        km, kv, _ = O.block_stats(kb, B)
        D = O.compensation_diag(qm, qv, km, kv, d)[0, 0]
        tok = np.array([[qi @ kj / math.sqrt(d) for kj in kb] for qi in qb])
        assert D == pytest.approx(tok.var(), rel=1e-12, abs=1e-13)
        # and the covariance is really diagonal
        cov = O.block_covariance(qb, B)[0]
        assert np.abs(cov - np.diag(np.diag(cov))).max() < 1e-12


def test_comp_exact_and_variance_identity_general():
    """General blocks: brute-force Var_{(i,j)}[lhat] equals
    (tr(SQ SK) + Qbar^T SK Qbar + Kbar^T SQ Kbar)/d (exact), which pins
    compensation_exact and the population moments; and the
    second-moment identity (1/(nq nk)) sum (dQ.dK)^2 = tr(SQ SK)."""
    for _ in range(30):
        d = int(RNG.integers(1, 9))
        nq, nk = int(RNG.integers(1, 12)), int(RNG.integers(1, 12))
        Qb, Kb = RNG.standard_normal((nq, d)) * 2 + 1, RNG.standard_normal((nk, d))
        qm, qv, _ = O.block_stats(Qb, nq)
        km, kv, _ = O.block_stats(Kb, nk)
        SQ, SK = O.block_covariance(Qb, nq)[0], O.block_covariance(Kb, nk)[0]
        ex = O.compensation_exact(SQ[None], SK[None], d)[0, 0]
        # brute-force trace
        tr = sum(SQ[s, t] * SK[t, s] for s in range(d) for t in range(d))
        assert ex == pytest.approx(tr / d, rel=1e-12, abs=1e-14)
        dq, dk = Qb - qm[0], Kb - km[0]
        sm = np.mean([(a @ b) ** 2 for a in dq for b in dk])
        assert sm == pytest.approx(tr, rel=1e-10, abs=1e-13)
        tok = np.array([[a @ b / math.sqrt(d) for b in Kb] for a in Qb])
        ident = (tr + qm[0] @ SK @ qm[0] + km[0] @ SQ @ km[0]) / d
        assert tok.var() == pytest.approx(ident, rel=1e-10, abs=1e-13)
        # diag compensation = the same identity with off-diagonals dropped
        Dd = O.compensation_diag(qm, qv, km, kv, d)[0, 0]
        dSQ, dSK = np.diag(np.diag(SQ)), np.diag(np.diag(SK))
        ident_d = (np.trace(dSQ @ dSK) + qm[0] @ dSK @ qm[0] + km[0] @ dSQ @ km[0]) / d
        assert Dd == pytest.approx(ident_d, rel=1e-12, abs=1e-14)
        assert Dd >= 0


def test_bound_U_sound():
    """Eq. logits-bound: max |lhat - l| <= U for every pair."""
    for sort in (False, True):
        X = RNG.standard_normal((64, 8)) * np.exp(RNG.normal(size=(64, 1)))
        Y = RNG.standard_normal((48, 8)) * np.exp(RNG.normal(size=(48, 1)))
        if sort:
            X, Y = X[O.norm_rank(X)], Y[O.norm_rank(Y)]
        U = O.deviation_bound(X, Y, 8)
        qm, _, _ = O.block_stats(X, 8)
        km, _, _ = O.block_stats(Y, 8)
        l = O.block_logits(qm, km, 8)
        tok = X @ Y.T / math.sqrt(8)
        for a, (s, e) in enumerate(O.make_grid(64, 8)):
            for b, (u, v) in enumerate(O.make_grid(48, 8)):
                assert np.abs(tok[s:e, u:v] - l[a, b]).max() <= U[a, b] + 1e-9


def test_bound_worked(golden):
    g = golden["bound_example"]
    U = (g["RQ"] * g["MK"] + g["MQ"] * g["RK"] + g["RQ"] * g["RK"]) / math.sqrt(g["d"])
    assert U == g["expected"]
    # deviation_bound on constant blocks is 0
    X = np.repeat(RNG.standard_normal((3, 4)), 4, axis=0)
    assert np.abs(O.deviation_bound(X, X, 4)).max() == 0


def test_max_logit_deviation_pins():
    """max_logit_deviation (the Fig. 2 ordinate) against: a worked
    example (d = 2: Q block {(1,0),(-1,0)}, K block {(2,0),(0,0)}: Qbar = 0, so l = 0
    and the extreme token logits are +-2/sqrt2 -> sqrt2; U = (1*2 + 1*1 + 1*1)/sqrt2
    = 2 sqrt2), the three-term decomposition of Eq. logit-deviation
    evaluated independently, U as an upper bound (Eq. logits-bound),
    constant blocks and B = 1 (tokens are their own blocks) -> 0."""
    X = np.array([[1.0, 0.0], [-1.0, 0.0]])
    Y = np.array([[2.0, 0.0], [0.0, 0.0]])
    assert abs(O.max_logit_deviation(X, Y, 2)[0, 0] - math.sqrt(2)) <= 1e-15
    assert abs(O.deviation_bound(X, Y, 2)[0, 0] - 2 * math.sqrt(2)) <= 1e-15
    for _ in range(5):
        d, B = 8, 8
        X = RNG.standard_normal((40, d)) * np.exp(RNG.normal(size=(40, 1)))
        Y = RNG.standard_normal((29, d)) * np.exp(RNG.normal(size=(29, 1)))
        dev = O.max_logit_deviation(X, Y, B)
        U = O.deviation_bound(X, Y, B)
        assert (dev <= U + 1e-12).all()
        for a, (s, e) in enumerate(O.make_grid(40, B)):
            for b, (u, v) in enumerate(O.make_grid(29, B)):
                qb, kb = X[s:e].mean(0), Y[u:v].mean(0)
                dq, dk = X[s:e] - qb, Y[u:v] - kb
                three = ((dq @ kb)[:, None] + (qb @ dk.T)[None, :] + dq @ dk.T) / math.sqrt(d)
                assert abs(np.abs(three).max() - dev[a, b]) <= 1e-12 * (1 + dev[a, b])
    C = np.repeat(RNG.standard_normal((3, 4)), 4, axis=0)
    assert np.abs(O.max_logit_deviation(C, C, 4)).max() <= 1e-14
    assert np.abs(O.max_logit_deviation(X, Y, 1)).max() <= 1e-12


# ---------------------------------------------------------------- budget and top-k
def test_kappa(golden):
    for rho, nk, exp in golden["kappa_configs"]["cases"]:
        assert O.kappa_from_density(rho, nk) == exp


@pytest.mark.parametrize("key", ["topk_a", "topk_tie"])
def test_topk_worked(golden, key):
    g = golden[key]
    mask, tau, idx = O.topk_mask(np.array([g["m"]]), g["kappa"])
    assert list(mask[0]) == g["expected_mask"]
    assert list(idx[0]) == [i for i, v in enumerate(g["expected_mask"]) if v]


def test_topk_brute_force():
    """Top-kappa = the kappa-subset of maximal mass (brute force, N_k <= 8)."""
    for _ in range(200):
        nk = int(RNG.integers(1, 9))
        kap = int(RNG.integers(1, nk + 1))
        m = O.softmax_rows(RNG.normal(size=(1, nk)))
        best = max(itertools.combinations(range(nk), kap), key=lambda c: sum(m[0, list(c)]))
        mask, tau, idx = O.topk_mask(m, kap)
        assert tuple(idx[0]) == best
        assert tau[0] == min(m[0, list(best)])
        assert mask.sum() == kap


def test_topk_monotone_in_density():
    m = O.softmax_rows(RNG.normal(size=(20, 50)))
    prev = None
    for rho in (0.02, 0.1, 0.3, 0.5, 0.8, 1.0):
        mask, _, _ = O.topk_mask(m, O.kappa_from_density(rho, 50))
        if prev is not None:
            assert (mask >= prev).all()
        prev = mask
    assert prev.all()


def test_topp_brute_force():
    """Reading A23: kappa_row is the minimum cardinality of ANY key-block subset
    whose mass reaches p, and the kept set is a maximum-mass subset of that
    size (so the greedy prefix is optimal) — brute force over all subsets,
    N_k <= 9, with and without the density cap."""
    for _ in range(150):
        nk = int(RNG.integers(1, 10))
        m = O.softmax_rows(RNG.normal(size=(1, nk)) * RNG.uniform(0.2, 3.0))
        p = float(RNG.uniform(0.05, 1.0))
        cap = int(RNG.integers(1, nk + 1))
        mask, tau, idx, kap = O.topp_mask(m, p, nk)
        sizes = [k for k in range(1, nk + 1)
                 if any(sum(m[0, list(c)]) >= p for c in itertools.combinations(range(nk), k))]
        kmin = sizes[0] if sizes else nk
        assert kap[0] == kmin
        best = max(sum(m[0, list(c)]) for c in itertools.combinations(range(nk), kmin))
        assert abs(m[0, idx[0]].sum() - best) <= 1e-15
        assert tau[0] == m[0, idx[0]].min()
        # capped: the kept set is top-min(kmin, cap) (same order as top-kappa)
        mask_c, _, idx_c, kap_c = O.topp_mask(m, p, cap)
        assert kap_c[0] == min(kmin, cap)
        assert list(idx_c[0]) == list(O.topk_mask(m, int(kap_c[0]))[2][0])


def test_topp_closed_forms():
    """Uniform rows: kappa_row = ceil(p N_k) (the mass of k blocks is k/N_k);
    p = 1 keeps every block with positive mass; a one-hot-dominant row keeps one
    block; kappa_row is non-decreasing in p."""
    for nk in (1, 3, 8, 50):
        m = np.full((1, nk), 1.0 / nk)
        for p in (0.1, 0.25, 0.5, 0.77, 1.0):
            # k/N_k >= p up to the fp64 rounding of the running sum (choose p off the grid)
            if abs(p * nk - round(p * nk)) < 1e-9:
                continue
            _, _, _, kap = O.topp_mask(m, p, nk)
            assert kap[0] == math.ceil(p * nk)
    m = np.array([[0.9, 0.05, 0.03, 0.02]])
    assert O.topp_mask(m, 0.9, 4)[3][0] == 1
    assert O.topp_mask(m, 0.95, 4)[3][0] == 2
    assert O.topp_mask(m, 1.0, 4)[3][0] == 4
    rows = O.softmax_rows(RNG.normal(size=(10, 40)) * 2)
    prev = np.zeros(10)
    for p in (0.1, 0.3, 0.5, 0.7, 0.9, 0.99):
        mask, _, _, kap = O.topp_mask(rows, p, 40)
        assert (kap >= prev).all() and (mask.sum(1) == kap).all()
        prev = kap


def test_topp_worked(golden):
    g = golden["topp_a"]
    mask, tau, idx, kap = O.topp_mask(np.array([g["m"]]), g["top_p"], len(g["m"]))
    assert list(mask[0]) == g["expected_mask"]
    assert kap[0] == sum(g["expected_mask"])


# ---------------------------------------------------------------- selection special cases
def test_constant_blocks_pooled_equals_oracle_map():
    """P:388 + Eq. oracle-dist: with constant, equal-size blocks
    Delta = 0 and m' = m = m_hat from the dense map (BJ pin)."""
    for seed in range(5):
        B, nb, d = 4, 6, 8
        Q, K, _ = constant_block_qkv(nb, B, d, seed=seed)
        sel = O.select_head(Q, K, B, 1.0, beta=1.0, sort=O.SORT_NONE, comp=O.COMP_DIAG)
        assert np.abs(sel.delta).max() == 0
        A = O.dense_attention_map(Q, K)
        mhat = O.oracle_block_mass(A, B, B)
        np.testing.assert_allclose(sel.m, mhat, atol=1e-12, rtol=0)


def test_singleton_blocks_m_equals_dense_map():
    """B = 1, sort none, comp none -> m' = A."""
    Q, K = RNG.standard_normal((9, 4)), RNG.standard_normal((7, 4))
    sel = O.select_head(Q, K, 1, 1.0, sort=O.SORT_NONE, comp=O.COMP_NONE)
    np.testing.assert_allclose(sel.m, O.dense_attention_map(Q, K), atol=1e-12, rtol=0)
    assert sel.mask.all()
    # and the oracle mass with B = 1 is A itself
    A = O.dense_attention_map(Q, K)
    np.testing.assert_allclose(O.oracle_block_mass(A, 1, 1), A, atol=1e-15)


def test_oracle_block_mass_rows_sum_to_one():
    Q, K = RNG.standard_normal((30, 4)), RNG.standard_normal((22, 4))
    mhat = O.oracle_block_mass(O.dense_attention_map(Q, K), 4, 5)
    np.testing.assert_allclose(mhat.sum(1), 1.0, atol=1e-12)


def test_select_pipeline_vs_straight_line():
    """select_head (Alg. 1 steps 1-10) equals a straight-line scalar
    re-derivation on a seed-fixed case, exercising the permutation,
    ragged stats, compensation sign and the softmax direction."""
    L, B, d = 37, 8, 16
    Q, K = RNG.standard_normal((L, d)) * 1.3, RNG.standard_normal((L, d))
    sel = O.select_head(Q, K, B, 0.4, beta=0.7, sort=O.SORT_QK, comp=O.COMP_DIAG)
    # straight line
    def keyf(r):
        return float(np.float32(sum(v * v for v in r)))
    pq = sorted(range(L), key=lambda i: (keyf(Q[i]), i))
    pk = sorted(range(L), key=lambda i: (keyf(K[i]), i))
    nb = (L + B - 1) // B
    def stats(X, p):
        ms, vs = [], []
        for g in range(nb):
            rows = [X[p[i]] for i in range(g * B, min((g + 1) * B, L))]
            mu = [sum(r[t] for r in rows) / len(rows) for t in range(d)]
            va = [sum((r[t] - mu[t]) ** 2 for r in rows) / len(rows) for t in range(d)]
            ms.append(mu)
            vs.append(va)
        return ms, vs
    qm, qv = stats(Q, pq)
    km, kv = stats(K, pk)
    for a in range(nb):
        lp = []
        for b in range(nb):
            l = sum(qm[a][t] * km[b][t] for t in range(d)) / math.sqrt(d)
            D = sum(qv[a][t] * km[b][t] ** 2 + kv[b][t] * qm[a][t] ** 2 + qv[a][t] * kv[b][t]
                    for t in range(d)) / d
            lp.append(l + 0.7 * D)
        mx = max(lp)
        ex = [math.exp(x - mx) for x in lp]
        m = [x / sum(ex) for x in ex]
        np.testing.assert_allclose(sel.m[a], m, atol=1e-13)
        kap = max(1, int(math.floor(0.4 * nb + 0.5)))
        chosen = sorted(sorted(range(nb), key=lambda j: (-m[j], j))[:kap])
        assert list(sel.kv_index[a]) == chosen
    assert list(sel.perm_q) == pq and list(sel.perm_k) == pk


# ---------------------------------------------------------------- attention
def test_dense_worked(golden):
    g = golden["dense_2x2"]
    out = O.dense_attention(np.array(g["Q"]), np.array(g["K"]), np.array(g["V"]))
    np.testing.assert_allclose(out, g["expected"], atol=g["tol"], rtol=0)


def test_dense_special_cases():
    K, V = RNG.standard_normal((1, 4)), RNG.standard_normal((1, 3))
    np.testing.assert_allclose(O.dense_attention(RNG.standard_normal((5, 4)), K, V), np.repeat(V, 5, 0), atol=1e-15)
    K, V = RNG.standard_normal((11, 4)), RNG.standard_normal((11, 3))
    np.testing.assert_allclose(O.dense_attention(np.zeros((2, 4)), K, V), np.repeat(V.mean(0, keepdims=True), 2, 0), atol=1e-14)


def test_dense_vs_triple_loop():
    Q, K, V = RNG.standard_normal((13, 5)), RNG.standard_normal((17, 5)), RNG.standard_normal((17, 3))
    out = O.dense_attention(Q, K, V, row_block=4)
    for i in range(13):
        s = [sum(Q[i, t] * K[j, t] for t in range(5)) / math.sqrt(5) for j in range(17)]
        mx = max(s)
        w = [math.exp(x - mx) for x in s]
        z = sum(w)
        for c in range(3):
            assert out[i, c] == pytest.approx(sum(w[j] * V[j, c] for j in range(17)) / z, abs=1e-12)


def _online_softmax_reference(Qs, Ks, Vs, kv_index, B, scale):
    """Independent brute force: per query row, streaming (online) softmax over
    the selected key blocks in pure Python."""
    L = Qs.shape[0]
    out = np.zeros((L, Vs.shape[1]))
    for i in range(L):
        g = i // B
        m, l = -math.inf, 0.0
        acc = np.zeros(Vs.shape[1])
        for j_blk in kv_index[g]:
            for j in range(j_blk * B, min((j_blk + 1) * B, Ks.shape[0])):
                s = float(Qs[i] @ Ks[j]) * scale
                mn = max(m, s)
                c = math.exp(m - mn) if m > -math.inf else 0.0
                p = math.exp(s - mn)
                l = l * c + p
                acc = acc * c + p * Vs[j]
                m = mn
        out[i] = acc / l
    return out


def test_sparse_vs_online_brute_force():
    for _ in range(10):
        L, B, d = int(RNG.integers(5, 40)), int(RNG.integers(2, 9)), 4
        N = (L + B - 1) // B
        Qs, Ks, Vs = RNG.standard_normal((L, d)), RNG.standard_normal((L, d)), RNG.standard_normal((L, 3))
        kap = int(RNG.integers(1, N + 1))
        idx = np.array([np.sort(RNG.choice(N, kap, replace=False)) for _ in range(N)])
        out, _ = O.block_sparse_attention_head(Qs, Ks, Vs, idx, B, 0.5)
        np.testing.assert_allclose(out, _online_softmax_reference(Qs, Ks, Vs, idx, B, 0.5), atol=1e-10, rtol=0)


def test_one_block_per_row_masked_softmax():
    L, B, d = 24, 4, 3
    Qs, Ks, Vs = RNG.standard_normal((L, d)), RNG.standard_normal((L, d)), RNG.standard_normal((L, d))
    idx = np.array([[(g * 5) % 6] for g in range(6)])
    out, _ = O.block_sparse_attention_head(Qs, Ks, Vs, idx, B, 1.0)
    for i in range(L):
        j0 = idx[i // B][0] * B
        s = Qs[i] @ Ks[j0:j0 + B].T
        w = np.exp(s - s.max())
        np.testing.assert_allclose(out[i], (w / w.sum()) @ Vs[j0:j0 + B], atol=1e-12)


def test_full_density_equals_dense_with_sorting():
    """0% sparsity reproduces dense attention (BJ), with sort = qk on the
    unsorted input — tests the permutation / un-permutation."""
    for cfg, L in (("T", 300), ("A", 200)):
        w = CONFIGS[cfg].with_(block_size=16, head_dim=32)
        q, k, v = make_qkv(w, seq_len=L, heads_q=2, heads_kv=1, special=False)
        p = O.Params(block_size=16, density=1.0, sort=O.SORT_QK)
        out, sels = O.ba_attention(q, k, v, p)
        for h in range(2):
            ref = O.dense_attention(q[0, h], k[0, 0], v[0, 0])
            np.testing.assert_allclose(out[0, h], ref, atol=1e-10, rtol=0)
            assert sels[(0, h)].mask.all()


def test_gqa_uses_group_kv_head():
    w = CONFIGS["C"].with_(block_size=8, head_dim=16)
    q, k, v = make_qkv(w, seq_len=40, heads_q=4, heads_kv=2, special=False)
    p = O.Params(block_size=8, density=1.0, sort=O.SORT_NONE)
    out, _ = O.ba_attention(q, k, v, p)
    for h in range(4):
        np.testing.assert_allclose(out[0, h], O.dense_attention(q[0, h], k[0, h // 2], v[0, h // 2]), atol=1e-10)


def test_sparse_flops_counting():
    # 50% on a 4x4 grid -> 8 pairs; L=256, B=16, kappa=4 -> 64 pairs
    idx = np.array([[0, 1]] * 4)
    assert O.sparse_flops(idx, 4 * 8, 4 * 8, 8, 2) == 8 * 2 * 8 * 8 * (2 + 2)
    idx = np.array([[0, 1, 2, 3]] * 16)
    assert O.sparse_flops(idx, 256, 256, 16, 1) == 64 * 2 * 16 * 16 * 2
    # ragged: last q block has 3 rows, last k block 3 cols
    idx = np.array([[2], [2], [2]])
    assert O.sparse_flops(idx, 19, 19, 8, 1) == 2 * (8 * 3 + 8 * 3 + 3 * 3) * 2
