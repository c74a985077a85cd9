"""Batch B = 2 (classifier-free guidance doubles the batch in the paper's models): every call indexes
(b, h) pairs correctly -- each batch entry reproduces the B = 1 result of its own data bit for bit
(statistics, fit, predict, attention, quantized attention, analysis metric)."""
import dataclasses

import numpy as np
import pytest
import torch

import synthetic as syn
from gpu_helpers import olayout

pytestmark = pytest.mark.gpu

W1 = syn.Workload("small-prefix", 1, 3, 128, 40, 3, 20, 19, 128)     # N=1180, ragged tail
W2 = dataclasses.replace(W1, batch=2)


def test_batch2_matches_two_batch1_runs():
    import paper_2601_11641_b200 as M
    P2, P1 = M.Plan(W2, top_k=5), M.Plan(W1, top_k=5)
    qa, ka, va = syn.family_s(W1, step=3, device="cuda")
    qb, kb, vb = syn.family_r(W1, device="cuda", seed=99)
    q, k, v = (torch.cat([x, y]).contiguous() for x, y in ((qa, qb), (ka, kb), (va, vb)))
    W = P2.collect_block_stats(q, k)
    X = P2.fit_mixture(W)
    keep = P2.keep_frames(X, X)
    rp, ci = P2.predict_block_mask(X * 0.5, X, 11, 12, 13, keep)
    o, lse = P2.block_sparse_attn_fwd(q, k, v, rp, ci)
    qbuf = P2.quantize_qkv(q, k, v)
    o8, l8 = P2.block_sparse_attn_fwd_q8(qbuf, rp, ci)
    rel = P2.map_rel_error(W, W.flip(0).contiguous())
    for b, (qq, kk, vv) in enumerate(((qa, ka, va), (qb, kb, vb))):
        Wb = P1.collect_block_stats(qq, kk)
        Xb = P1.fit_mixture(Wb)
        keepb = P1.keep_frames(Xb, Xb)
        rpb, cib = P1.predict_block_mask(Xb * 0.5, Xb, 11, 12, 13, keepb)
        ob, lb = P1.block_sparse_attn_fwd(qq, kk, vv, rpb, cib)
        o8b, l8b = P1.block_sparse_attn_fwd_q8(P1.quantize_qkv(qq, kk, vv), rpb, cib)
        assert torch.equal(W[b], Wb[0]) and torch.equal(X[b], Xb[0]) and torch.equal(keep[b], keepb[0])
        assert torch.equal(rp[b], rpb[0])
        for h in range(W1.heads):
            nnz = int(rpb[0, h, -1])
            assert torch.equal(ci[b, h, :nnz], cib[0, h, :nnz])
        assert torch.equal(o[b], ob[0]) and torch.equal(lse[b], lb[0])
        assert torch.equal(o8[b], o8b[0]) and torch.equal(l8[b], l8b[0])
    assert torch.all(rel >= 0)
