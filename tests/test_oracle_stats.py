"""Pins for oracle O2 (pooled statistic) and O2' (Eq. 2 sparsity) -- no GPU.

O2 has no paper anchor (north-star construct, "parity unpinned" vs the paper); it is pinned here
by identities: z_ij equals the block mean of the token scores s Q_p . K_q (brute force), rows of
W sum to 1, the closed form for block-constant Q/K, and the uniform case Q = 0.
O2' is pinned by SPEC.md S:106-111 examples and monotonicity in eta.
"""
import math

import numpy as np
import torch

import oracle as O


def _lay():
    return O.make_layout(1, 2, 8, 3, 3, 2, 5, 4)     # N = 33, ragged last block, prefix


def test_pooled_z_is_block_mean_of_token_scores():
    L = _lay()
    g = torch.Generator().manual_seed(0)
    q = torch.randn((1, 2, L.N, 8), generator=g, dtype=torch.float64)
    k = torch.randn((1, 2, L.N, 8), generator=g, dtype=torch.float64)
    W, z = O.pooled_block_stats(q, k, L, return_z=True)
    s = 1 / math.sqrt(8)
    qn, kn = q.numpy(), k.numpy()
    for h in range(2):
        T = s * qn[0, h] @ kn[0, h].T
        for i in range(L.n):
            for j in range(L.n):
                (a, b), (c, d) = L.block_range(i), L.block_range(j)
                assert abs(T[a:b, c:d].mean() - z[0, h, i, j]) <= 1e-13
    assert np.allclose(W.sum(-1), 1.0, atol=1e-14)


def test_pooled_closed_form_constant_blocks():
    L = _lay()
    rng = np.random.default_rng(1)
    qb, kb = rng.standard_normal((L.n, 8)), rng.standard_normal((L.n, 8))
    tb = np.arange(L.N) // L.block
    q = np.broadcast_to(qb[tb], (1, 2, L.N, 8)).copy()
    k = np.broadcast_to(kb[tb], (1, 2, L.N, 8)).copy()
    W = O.pooled_block_stats(q, k, L)
    sizes = np.array([L.block_size(i) for i in range(L.n)])
    # every token pair (p,q) in block (i,j) scores s qb_i . kb_j: softmax mass of block j
    for i in range(L.n):
        e = sizes * np.exp(qb[i] @ kb.T / math.sqrt(8))
        assert np.allclose(W[0, 0, i], e / e.sum(), atol=1e-14)


def test_pooled_uniform_when_q_zero():
    L = _lay()
    q = np.zeros((1, 2, L.N, 8))
    k = np.random.default_rng(2).standard_normal((1, 2, L.N, 8))
    W = O.pooled_block_stats(q, k, L)
    sizes = np.array([L.block_size(i) for i in range(L.n)])
    assert np.allclose(W, sizes / L.N, atol=1e-15)


def test_sparsity_spec_examples():
    L = O.make_layout(1, 1, 8, 0, 1, 1, 256, 128)
    assert np.array_equal(O.sparsity_from_map(np.zeros((256, 256)), L), np.ones((2, 2)))
    assert np.array_equal(O.sparsity_from_map(np.ones((256, 256)), L), np.zeros((2, 2)))
    L4 = O.make_layout(1, 1, 8, 0, 1, 1, 4, 2)
    A = np.ones((4, 4))
    A[0, 0] = A[0, 1] = 0.0
    A[1, 0], A[1, 1] = 0.5, 0.5
    assert O.sparsity_from_map(A, L4)[0, 0] == 0.5


def test_sparsity_monotone_in_eta():
    L = _lay()
    rng = np.random.default_rng(3)
    q = rng.standard_normal((1, 2, L.N, 8)) * 2
    k = rng.standard_normal((1, 2, L.N, 8)) * 2
    prev = None
    for eta in (1e-6, 1e-4, 1e-2, 1e-1):
        S = O.exact_sparsity(q, k, L, eta)
        assert np.all((S >= 0) & (S <= 1))
        if prev is not None:
            assert np.all(prev <= S)
        prev = S


def test_masked_exact_sparsity_all_ones_equals_dense():
    L = _lay()
    rng = np.random.default_rng(4)
    q = rng.standard_normal((1, 2, L.N, 8)) * 2
    k = rng.standard_normal((1, 2, L.N, 8)) * 2
    ones = np.ones((1, 2, L.n, L.n), dtype=bool)
    Sm, lse = O.exact_sparsity_masked(q, k, ones, L, 1e-3)
    assert np.array_equal(Sm, O.exact_sparsity(q, k, L, 1e-3))
    from scipy.special import logsumexp
    assert np.allclose(lse, logsumexp(q @ np.swapaxes(k, -1, -2) / np.sqrt(8), axis=-1), atol=1e-12)


def test_masked_exact_sparsity_renormalises_over_selection():
    L = _lay()
    rng = np.random.default_rng(5)
    q = rng.standard_normal((1, 1, L.N, 8))
    k = rng.standard_normal((1, 1, L.N, 8))
    m = np.zeros((1, 1, L.n, L.n), dtype=bool)
    m[0, 0, :, 0] = True                     # a single key block per row: uniform-ish P over it
    Sm, _ = O.exact_sparsity_masked(q, k, m, L, 1e-9)
    assert np.all(np.isnan(Sm[0, 0, :, 1:]))
    assert np.all(Sm[0, 0, :, 0] == 0.0)     # no probability over a single 4-key block falls below 1e-9


def test_masked_exact_sparsity_rows_match_the_whole_map():
    """The row-sampled form (used for full-size GPU checks) restricts the same Eq. 2 computation."""
    L = _lay()
    rng = np.random.default_rng(6)
    q = rng.standard_normal((1, 2, L.N, 8)) * 1.5
    k = rng.standard_normal((1, 2, L.N, 8)) * 1.5
    m = rng.random((1, 2, L.n, L.n)) < 0.5
    m[0, 1, 2] = True
    Sm, lse = O.exact_sparsity_masked(q, k, m, L, 1e-2)
    rows = O.exact_sparsity_masked_rows(q, k, m[0, 1], L, 0, 1, range(L.n), 1e-2)
    for i, (row, lse_i) in rows.items():
        lo, hi = L.block_range(i)
        assert np.array_equal(np.isnan(row), np.isnan(Sm[0, 1, i]))
        assert np.allclose(row[~np.isnan(row)], Sm[0, 1, i][~np.isnan(row)], atol=0)
        if m[0, 1, i].any():
            assert np.allclose(lse_i, lse[0, 1, lo:hi], atol=1e-12)


# ------------------------------------------------------------------------------------------------
# Brute-force pins for O2' (Eq. 2, on the POST-softmax map of Alg. 1 line 5):
# pure-Python loops over single tokens (math.exp, explicit per-row normalisation, strict "<"),
# independent of the numpy code in oracle/stats.py.  A dropped row normalisation, a "<=" for "<",
# a transposed operand or a mask applied before/after the normalisation fails one of them.

def _bf_row_probs(qrow, krows, s, allowed):
    """softmax over the allowed keys of one query row, by explicit loops."""
    logits = [s * sum(a * b for a, b in zip(qrow, kr)) if ok else None for kr, ok in zip(krows, allowed)]
    mx = max(x for x in logits if x is not None)
    e = [math.exp(x - mx) if x is not None else None for x in logits]
    z = sum(x for x in e if x is not None)
    return [x / z if x is not None else None for x in e], mx + math.log(z)


def _bf_sparsity(q, k, L, eta, block_mask=None):
    """Eq. 2 by enumeration: S_ij = #{(p,q) in I_i x I_j : P_pq < eta} / (|I_i||I_j|)."""
    B, H, N, D = q.shape
    s = 1.0 / math.sqrt(D)
    S = np.full((B, H, L.n, L.n), np.nan)
    lse = np.zeros((B, H, N))
    blk = [p // L.block for p in range(N)]
    for b in range(B):
        for h in range(H):
            cnt = np.zeros((L.n, L.n))
            for p in range(N):
                allowed = [True] * N if block_mask is None else [bool(block_mask[b, h, blk[p], blk[t]]) for t in range(N)]
                P, lse[b, h, p] = _bf_row_probs(q[b, h, p], k[b, h], s, allowed)
                for t in range(N):
                    if P[t] is not None and P[t] < eta:
                        cnt[blk[p], blk[t]] += 1
            for i in range(L.n):
                for j in range(L.n):
                    if block_mask is None or block_mask[b, h, i, j]:
                        S[b, h, i, j] = cnt[i, j] / (L.block_size(i) * L.block_size(j))
    return S, lse


def test_exact_sparsity_brute_force_ragged():
    L = O.make_layout(1, 2, 4, 3, 2, 2, 5, 4)       # N = 23: prefix block + ragged last block (size 3)
    rng = np.random.default_rng(11)
    q = rng.standard_normal((1, 2, L.N, 4)) * 2.5
    k = rng.standard_normal((1, 2, L.N, 4)) * 2.5
    for eta in (1e-3, 2e-2, 0.05):
        S_bf, _ = _bf_sparsity(q, k, L, eta)
        assert np.allclose(O.exact_sparsity(q, k, L, eta), S_bf, atol=1e-15, rtol=0)
        assert 0 < np.nanmean(S_bf) < 1                 # the case is not degenerate


def test_exact_sparsity_masked_brute_force_ragged():
    L = O.make_layout(1, 2, 4, 3, 2, 2, 5, 4)
    rng = np.random.default_rng(12)
    q = rng.standard_normal((1, 2, L.N, 4)) * 2.5
    k = rng.standard_normal((1, 2, L.N, 4)) * 2.5
    m = rng.random((1, 2, L.n, L.n)) < 0.5
    m[..., np.arange(L.n), np.arange(L.n)] = True
    S_bf, lse_bf = _bf_sparsity(q, k, L, 2e-2, m)
    Sm, lse = O.exact_sparsity_masked(q, k, m, L, 2e-2)
    assert np.array_equal(np.isnan(Sm), np.isnan(S_bf))
    assert np.allclose(Sm[~np.isnan(Sm)], S_bf[~np.isnan(S_bf)], atol=1e-15, rtol=0)
    assert np.allclose(lse, lse_bf, atol=1e-12)
    rows = O.exact_sparsity_masked_rows(q, k, m[0, 1], L, 0, 1, range(L.n), 2e-2)
    for i, (row, lse_i) in rows.items():
        ok = ~np.isnan(S_bf[0, 1, i])
        assert np.array_equal(np.isnan(row), ~ok)
        assert np.allclose(row[ok], S_bf[0, 1, i][ok], atol=1e-15, rtol=0)


def test_exact_sparsity_strict_threshold_on_exact_probabilities():
    """Q = 0 makes every post-softmax row uniform: P = 1/N exactly when N is a power of two.
    eta = 1/N must count nothing (strict "<") and the next double up must count everything;
    an unnormalised map (P = 1) would count nothing for both."""
    L = O.make_layout(1, 1, 4, 0, 2, 4, 4, 8)            # N = 32, n = 4
    q = np.zeros((1, 1, 32, 4))
    k = np.random.default_rng(13).standard_normal((1, 1, 32, 4))
    eta = 1.0 / 32
    assert np.all(O.exact_sparsity(q, k, L, eta) == 0.0)
    assert np.all(O.exact_sparsity(q, k, L, np.nextafter(eta, 1.0)) == 1.0)
    # masked form: two selected key blocks of 8 -> P = 1/16 exactly over the selection
    m = np.zeros((1, 1, L.n, L.n), dtype=bool)
    m[0, 0, :, 1] = m[0, 0, :, 3] = True
    Sm, lse = O.exact_sparsity_masked(q, k, m, L, 1.0 / 16)
    assert np.all(Sm[m] == 0.0) and np.all(np.isnan(Sm[~m]))
    Sm, _ = O.exact_sparsity_masked(q, k, m, L, np.nextafter(1.0 / 16, 1.0))
    assert np.all(Sm[m] == 1.0)
    assert np.allclose(lse, math.log(16), atol=1e-15)
    rows = O.exact_sparsity_masked_rows(q, k, m[0, 0], L, 0, 0, range(L.n), 1.0 / 16)
    assert all(np.all(r[~np.isnan(r)] == 0.0) for r, _ in rows.values())
