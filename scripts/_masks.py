"""Structured block masks for the bring-up timing scripts, built by the library's own predictor
(K2b) from seeded random intensities: a random Top-K of the diagonal / column patterns plus ~70 %
of the frame squares -- the same kind of mask the pipeline produces.  (No oracle code here: only
tests/, smoke() and bench.py's CPU legs use oracle/.)"""
import torch

import synthetic as syn


def structured_csr(P, w, seed: int = 0, top_k=None, keep_frac: float = 0.7):
    n = P.n
    x = syn.random_intensities(w.batch, w.heads, P.p, seed=seed, device="cuda")
    g = torch.Generator().manual_seed(seed + 1)
    keep = (torch.rand((w.batch, w.heads, w.frames), generator=g) < keep_frac).to(torch.uint8).cuda()
    rp, ci = P.predict_block_mask(x, x, 11, 12, 13, keep, top_k=top_k or max(4, n // 12))
    torch.cuda.synchronize()
    return rp, ci
