"""O9 -- masked softmax attention (oracle; test infrastructure only).

Full attention (§3): O_h = softmax(Q_h K_h^T / sqrt(d)) V_h.
Sparse attention (§3 Eq. 1): SA = softmax(A + M) V, M in {-inf, 0}^{N x N}, with the
block mask upsampled to tokens (Alg. 1).  For token p of query block i:
  O_p = sum_{q in K(i)} softmax_q(s Q_p . K_q) V_q,   K(i) = union of I_j over passing j,
  lse_p = ln sum_{q in K(i)} exp(s Q_p . K_q).
Reading Z15: an empty K(i) gives O_p = 0 and lse_p = -inf.
Evaluated in fp64 from the (bf16) inputs with max-subtraction.
"""
from __future__ import annotations

import numpy as np

from .layout import Layout
from .stats import _f64


def _rows_attention(qr, k, v, keymask, s):
    """qr [R,D], k,v [N,D], keymask [R,N] bool -> O [R,D], lse [R]."""
    A = s * (qr @ k.T)
    A = np.where(keymask, A, -np.inf)
    m = A.max(axis=1, keepdims=True)
    empty = ~np.isfinite(m[:, 0])
    m = np.where(np.isfinite(m), m, 0.0)
    e = np.exp(A - m)
    l = e.sum(axis=1, keepdims=True)
    with np.errstate(invalid="ignore", divide="ignore"):
        O = (e @ v) / l
        lse = m[:, 0] + np.log(l[:, 0])
    O[empty] = 0.0
    lse[empty] = -np.inf
    return O, lse


def masked_attention_rows(q, k, v, mask, L: Layout, b: int, h: int, qblocks, scale=None):
    """O, lse for the query blocks ``qblocks`` of head (b,h); mask is that head's n x n block mask."""
    s = 1.0 / np.sqrt(L.head_dim) if not scale else float(scale)
    qh = _f64(q[b, h]) if not isinstance(q, np.ndarray) else q[b, h]
    kh = _f64(k[b, h]) if not isinstance(k, np.ndarray) else k[b, h]
    vh = _f64(v[b, h]) if not isinstance(v, np.ndarray) else v[b, h]
    N = L.N
    tok_block = np.arange(N) // L.block
    outs, lses = [], []
    for i in qblocks:
        lo, hi = L.block_range(i)
        keymask = np.broadcast_to(mask[i][tok_block], (hi - lo, N))
        O, lse = _rows_attention(qh[lo:hi], kh, vh, keymask, s)
        outs.append(O)
        lses.append(lse)
    return outs, lses


def masked_attention(q, k, v, masks, L: Layout, scale=None):
    """O [B,H,N,D], lse [B,H,N] for per-head block masks [B,H,n,n] (tiny shapes)."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    B, H, N, D = q.shape
    O = np.zeros((B, H, N, D))
    lse = np.zeros((B, H, N))
    for b in range(B):
        for h in range(H):
            outs, lses = masked_attention_rows(q, k, v, masks[b, h], L, b, h, range(L.n), scale)
            for i, (o, l_) in enumerate(zip(outs, lses)):
                lo, hi = L.block_range(i)
                O[b, h, lo:hi] = o
                lse[b, h, lo:hi] = l_
    return O, lse


def dense_attention(q, k, v, scale=None):
    """Full attention (§3) in fp64, [B,H,N,D]."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    D = q.shape[-1]
    s = 1.0 / np.sqrt(D) if not scale else float(scale)
    A = s * np.einsum("bhpd,bhqd->bhpq", q, k)
    A = np.exp(A - A.max(axis=-1, keepdims=True))
    A /= A.sum(axis=-1, keepdims=True)
    return np.einsum("bhpq,bhqd->bhpd", A, v)
