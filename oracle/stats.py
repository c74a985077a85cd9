"""O2 / O2' -- block statistics (oracle; test infrastructure only).

O2' EXACT (§4.1 Eq. 2): S_(i,j) = (1/B^2) sum_{x,y} 1(A_(iB+x, jB+y) < eta),
   with A the post-softmax attention map (reading Z2, Alg. 1 P:995 "A = softmax(QK^T/sqrt d)"),
   strict "<", eta = 1e-4 (App. A).  Ragged blocks divide by |I_i||I_j| (Z16).
   Informativeness polarity (reading Z3): U = -S ("less S = more informative"), so that the
   paper's ascending Top-K on fit(S) is the descending Top-K on fit(U) = -fit(S) exactly.

O2 POOLED (BASELINE.json north_star (1); the hot-path substitute for Eq. 2, reading Z1):
   qbar_i = mean_{p in I_i} Q_p, kbar_j likewise; z_ij = s * qbar_i . kbar_j, s = 1/sqrt(D)
   (P:106); W_ij = |I_j| e^{z_ij} / sum_j' |I_j'| e^{z_ij'}  (block mass of the pooled
   surrogate: every key of block j scores z_ij).  U = W.
   -- parity unpinned against the paper (north-star construct); pinned by identities in
   tests/test_oracle_stats.py.
"""
from __future__ import annotations

import numpy as np

from .layout import Layout


def _f64(x):
    import torch
    if isinstance(x, torch.Tensor):
        return x.detach().to("cpu", dtype=torch.float64).numpy()
    return np.asarray(x, dtype=np.float64)


def pooled_block_stats(q, k, L: Layout, scale: float | None = None, return_z: bool = False):
    """POOLED statistic W [B,H,n,n] (fp64) from Q, K [B,H,N,D]."""
    q = _f64(q)
    k = _f64(k)
    s = 1.0 / np.sqrt(L.head_dim) if not scale else float(scale)
    n = L.n
    sizes = np.array([L.block_size(i) for i in range(n)], dtype=np.float64)
    B, H = q.shape[0], q.shape[1]
    qbar = np.empty((B, H, n, L.head_dim))
    kbar = np.empty((B, H, n, L.head_dim))
    for i in range(n):
        lo, hi = L.block_range(i)
        qbar[:, :, i] = q[:, :, lo:hi].mean(axis=2)
        kbar[:, :, i] = k[:, :, lo:hi].mean(axis=2)
    z = s * np.einsum("bhid,bhjd->bhij", qbar, kbar)
    logits = z + np.log(sizes)[None, None, None, :]
    m = logits.max(axis=-1, keepdims=True)
    e = np.exp(logits - m)
    W = e / e.sum(axis=-1, keepdims=True)
    return (W, z) if return_z else W


def exact_sparsity(q, k, L: Layout, eta: float = 1e-4, scale: float | None = None):
    """EXACT Eq. 2 sparsity map S [B,H,n,n] from the full post-softmax map (tiny shapes only)."""
    q = _f64(q)
    k = _f64(k)
    s = 1.0 / np.sqrt(L.head_dim) if not scale else float(scale)
    B, H, N, _ = q.shape
    n = L.n
    S = np.zeros((B, H, n, n))
    for b in range(B):
        for h in range(H):
            A = s * q[b, h] @ k[b, h].T
            A = np.exp(A - A.max(axis=1, keepdims=True))
            A /= A.sum(axis=1, keepdims=True)                      # P:995 post-softmax map
            S[b, h] = sparsity_from_map(A, L, eta)
    return S


def sparsity_from_map(A, L: Layout, eta: float = 1e-4):
    """Eq. 2 on one N x N attention map: fraction of entries strictly below eta per block."""
    A = np.asarray(A, dtype=np.float64)
    n = L.n
    below = (A < eta)
    S = np.zeros((n, n))
    for i in range(n):
        ilo, ihi = L.block_range(i)
        for j in range(n):
            jlo, jhi = L.block_range(j)
            S[i, j] = below[ilo:ihi, jlo:jhi].sum() / ((ihi - ilo) * (jhi - jlo))
    return S


def informativeness_from_sparsity(S):
    """Reading Z3: U = -S (larger = more informative; fit(U) = -fit(S), so descending on fit(U) is the
    paper's ascending-on-fit(S) Top-K of P:437 with no per-family offset)."""
    return -np.asarray(S, dtype=np.float64)


def exact_sparsity_masked(q, k, masks, L: Layout, eta: float = 1e-4, scale: float | None = None):
    """Eq. 2 on the MASKED post-softmax map of sparse attention (Eq. 1; Eq. 5's A_masked with
    reading Z12: normalised over the unmasked keys only).  Returns S [B,H,n,n] with NaN at the blocks
    the mask removes (they keep their history in Eq. 5) and the log-sum-exp lse [B,H,N] of each row
    over its unmasked keys."""
    q = _f64(q)
    k = _f64(k)
    masks = np.asarray(masks, dtype=bool)
    s = 1.0 / np.sqrt(L.head_dim) if not scale else float(scale)
    B, H, N, _ = q.shape
    n = L.n
    tb = np.arange(N) // L.block
    S = np.full((B, H, n, n), np.nan)
    lse = np.zeros((B, H, N))
    for b in range(B):
        for h in range(H):
            A = s * q[b, h] @ k[b, h].T
            km = masks[b, h][tb][:, tb]
            A = np.where(km, A, -np.inf)
            m = A.max(axis=1, keepdims=True)
            e = np.exp(A - m)
            z = e.sum(axis=1, keepdims=True)
            lse[b, h] = (m + np.log(z))[:, 0]
            P = e / z                                              # masked, renormalised (Z12)
            for i in range(n):
                ilo, ihi = L.block_range(i)
                for j in np.nonzero(masks[b, h, i])[0]:
                    jlo, jhi = L.block_range(j)
                    S[b, h, i, j] = (P[ilo:ihi, jlo:jhi] < eta).sum() / ((ihi - ilo) * (jhi - jlo))
    return S, lse


def exact_sparsity_masked_rows(q, k, mask, L: Layout, b: int, h: int, qblocks, eta: float = 1e-4,
                               scale: float | None = None):
    """exact_sparsity_masked for the query blocks ``qblocks`` of one (b, h) only (the same Eq. 2 on the
    masked, renormalised map, row block by row block), so that full-size layouts can be checked on
    samples.  ``mask`` is that head's n x n block mask.  Returns {i: (S_row [n] with NaN off the mask,
    lse [|I_i|])}."""
    q = _f64(q)[b, h]
    k = _f64(k)[b, h]
    mask = np.asarray(mask, dtype=bool)
    s = 1.0 / np.sqrt(L.head_dim) if not scale else float(scale)
    N = q.shape[0]
    tb = np.arange(N) // L.block
    out = {}
    for i in qblocks:
        ilo, ihi = L.block_range(i)
        A = s * q[ilo:ihi] @ k.T
        A = np.where(mask[i][tb][None, :], A, -np.inf)
        m = A.max(axis=1, keepdims=True)
        e = np.exp(A - m)
        z = e.sum(axis=1, keepdims=True)
        P = e / z
        row = np.full(L.n, np.nan)
        for j in np.nonzero(mask[i])[0]:
            jlo, jhi = L.block_range(j)
            row[j] = (P[:, jlo:jhi] < eta).sum() / ((ihi - ilo) * (jhi - jlo))
        out[int(i)] = (row, (m + np.log(z))[:, 0])
    return out
