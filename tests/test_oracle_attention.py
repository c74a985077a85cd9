"""Pins for oracle O9 (masked softmax attention) -- no GPU.

All-ones mask == dense softmax attention (north star), single-entry rows return the V
row, a -1e9 dense reference, pure-Python brute force on tiny inputs, and the
empty-row convention (reading Z15).
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synthetic as syn


def _lay(N_frames=4, hw=8, b=4, D=8, P0=0):
    return O.make_layout(1, 2, D, P0, N_frames, 1, hw, b)


def _qkv(L, seed=0):
    g = torch.Generator().manual_seed(seed)
    sh = (L.batch, L.heads, L.N, L.head_dim)
    return [torch.randn(sh, generator=g, dtype=torch.float64).numpy() for _ in range(3)]


def test_all_ones_mask_is_dense_attention():
    L = _lay()
    q, k, v = _qkv(L)
    ones = np.ones((1, 2, L.n, L.n), dtype=bool)
    O1, lse = O.masked_attention(q, k, v, ones, L)
    assert np.max(np.abs(O1 - O.dense_attention(q, k, v))) <= 1e-12
    s = 1 / math.sqrt(L.head_dim)
    A = s * np.einsum("bhpd,bhqd->bhpq", q, k)
    from scipy.special import logsumexp
    assert np.max(np.abs(lse - logsumexp(A, axis=-1))) <= 1e-12


def test_tiny_config_all_ones_is_dense():
    L = O.make_layout(*[getattr(syn.TINY, f) for f in
                        ("batch", "heads", "head_dim", "prefix_tokens", "frames", "height", "width", "block")])
    q, k, v = syn.family_r(syn.TINY)
    ones = np.ones((1, 2, L.n, L.n), dtype=bool)
    O1, _ = O.masked_attention(q, k, v, ones, L)
    assert np.max(np.abs(O1 - O.dense_attention(q, k, v))) <= 1e-12


def test_single_entry_rows_return_v():
    L = O.make_layout(1, 1, 4, 0, 1, 1, 6, 1)      # block = 1 token
    q, k, v = _qkv(L, 1)
    m = np.eye(L.n, dtype=bool)[None, None]
    O1, _ = O.masked_attention(q, k, v, m, L)
    assert np.allclose(O1, v, atol=1e-15)


def test_matches_minus_1e9_dense_reference():
    L = _lay(b=2)
    q, k, v = _qkv(L, 2)
    rng = np.random.default_rng(3)
    m = rng.random((1, 2, L.n, L.n)) < 0.5
    m |= np.eye(L.n, dtype=bool)
    O1, _ = O.masked_attention(q, k, v, m, L)
    s = 1 / math.sqrt(L.head_dim)
    tb = np.arange(L.N) // L.block
    for h in range(2):
        A = s * q[0, h] @ k[0, h].T
        A = np.where(m[0, h][tb][:, tb], A, A - 1e9)
        P = np.exp(A - A.max(1, keepdims=True))
        P /= P.sum(1, keepdims=True)
        assert np.allclose(P.sum(1), 1.0, atol=1e-14)         # probability rows sum to 1
        assert np.max(np.abs(P @ v[0, h] - O1[0, h])) <= 1e-9


def test_brute_force_python_loops():
    L = O.make_layout(1, 1, 3, 1, 2, 1, 3, 2)       # N = 7, ragged blocks, prefix
    q, k, v = _qkv(L, 4)
    m = np.array([[1, 0, 1, 0], [0, 1, 0, 0], [1, 1, 0, 1], [0, 0, 0, 1]], dtype=bool)[None, None]
    O1, lse = O.masked_attention(q, k, v, m, L)
    s = 1 / math.sqrt(3)
    for p in range(L.N):
        keys = [t for t in range(L.N) if m[0, 0, p // 2, t // 2]]
        sc = [s * sum(q[0, 0, p, d] * k[0, 0, t, d] for d in range(3)) for t in keys]
        mx = max(sc)
        w = [math.exp(x - mx) for x in sc]
        z = sum(w)
        for d in range(3):
            ref = sum(wi * v[0, 0, t, d] for wi, t in zip(w, keys)) / z
            assert abs(O1[0, 0, p, d] - ref) <= 1e-12
        assert abs(lse[0, 0, p] - (mx + math.log(z))) <= 1e-12


def test_empty_row_convention():
    L = _lay()
    q, k, v = _qkv(L, 5)
    m = np.ones((1, 2, L.n, L.n), dtype=bool)
    m[0, 1, 2, :] = False
    O1, lse = O.masked_attention(q, k, v, m, L)
    lo, hi = L.block_range(2)
    assert np.all(O1[0, 1, lo:hi] == 0) and np.all(np.isneginf(lse[0, 1, lo:hi]))
