"""GPU parity of the analysis metrics through the C ABI against the fp64 oracle.

Tolerance: both sides accumulate fp32 maps / fp64 intensities in fp64; they differ only in summation
order, so 1e-12 relative."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synthetic as syn
from gpu_helpers import masks_to_csr, olayout

pytestmark = pytest.mark.gpu

COG_SMALL = syn.Workload("cog-small", 1, 2, 64, 226, 3, 30, 45, 128)
WORKLOADS = [syn.TINY, COG_SMALL, syn.COGVIDEOX]


@pytest.fixture(scope="module")
def M():
    import paper_2601_11641_b200 as m
    return m


@pytest.mark.parametrize("w", WORKLOADS, ids=lambda w: w.name)
def test_map_rel_error_parity(M, w):
    L = olayout(w)
    P = M.Plan(w)
    A = syn.random_stats(w.batch, w.heads, L.n, seed=31, device="cuda")
    B = syn.random_stats(w.batch, w.heads, L.n, seed=32, device="cuda")
    out = P.map_rel_error(A, B)
    out2 = P.map_rel_error(A, B)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)                                     # deterministic
    An, Bn = A.double().cpu().numpy(), B.double().cpu().numpy()
    for b in range(w.batch):
        for h in range(w.heads):
            assert out[b, h].item() == pytest.approx(O.rel_frobenius(An[b, h], Bn[b, h]), rel=1e-12)


def test_map_rel_error_degenerate(M):
    w = syn.TINY
    L = olayout(w)
    P = M.Plan(w)
    A = syn.random_stats(w.batch, w.heads, L.n, seed=33, device="cuda")
    Z = torch.zeros_like(A)
    assert torch.all(P.map_rel_error(A, A) == 0)
    assert torch.all(P.map_rel_error(Z, Z) == 0)
    assert torch.all(torch.isinf(P.map_rel_error(A, Z)))
    with pytest.raises(ValueError):
        P.map_rel_error(A.double(), A)


@pytest.mark.parametrize("w", WORKLOADS, ids=lambda w: w.name)
def test_linearity_nre_parity(M, w):
    L = olayout(w)
    P = M.Plan(w)
    xp = syn.random_intensities(w.batch, w.heads, L.p, seed=41, device="cuda")
    xc = syn.random_intensities(w.batch, w.heads, L.p, seed=42, device="cuda")
    ts = list(range(23, 33))
    traj = torch.stack([syn.random_intensities(w.batch, w.heads, L.p, seed=50 + s, device="cuda") for s in range(10)])
    traj[:, :, :, 0] = 1.25                                           # flat pattern -> NaN
    out = P.linearity_nre(xp, xc, 12, 22, traj.contiguous(), ts).cpu().numpy()
    tn, xpn, xcn = traj.cpu().numpy(), xp.cpu().numpy(), xc.cpu().numpy()
    for b in range(w.batch):
        for h in range(w.heads):
            ref = O.linearity_nre(xpn[b, h], xcn[b, h], 12, 22, tn[:, b, h], ts, L)
            assert np.array_equal(np.isnan(out[b, h]), np.isnan(ref))
            ok = ~np.isnan(ref)
            assert np.allclose(out[b, h][ok], ref[ok], rtol=1e-12, atol=0)


def test_linearity_nre_errors(M):
    w = syn.TINY
    L = olayout(w)
    P = M.Plan(w)
    x = syn.random_intensities(w.batch, w.heads, L.p, seed=43, device="cuda")
    traj = x[None].contiguous()
    with pytest.raises(M.ModditError, match="t_prev == t_curr"):
        P.linearity_nre(x, x, 5, 5, traj, [6])
    with pytest.raises(M.ModditError, match="S = 0|non-NULL"):   # an empty trajectory has no storage
        P.linearity_nre(x, x, 4, 5, x[:0][None].reshape(0, *x.shape).contiguous(), [])
    many = x[None].expand(65, *x.shape).contiguous()
    with pytest.raises(M.ModditError, match="S = 65"):
        P.linearity_nre(x, x, 4, 5, many, list(range(65)))


def test_reconstruction_nre_of_the_gpu_update(M):
    """NRE(t) of Eq. 5 as the pipeline runs it: history after mod_update_online_mask vs the fresh map
    (ground truth); without renormalisation it equals the oracle's brute-force value."""
    w = COG_SMALL
    L = olayout(w)
    P = M.Plan(w, masked_renorm=False)
    gt = syn.random_stats(w.batch, w.heads, L.n, seed=61, device="cuda")
    hist = syn.random_stats(w.batch, w.heads, L.n, seed=62, device="cuda")
    masks = np.random.default_rng(63).random((w.batch, w.heads, L.n, L.n)) < 0.35
    rp, ci = masks_to_csr(masks)
    h0 = hist.double().cpu().numpy()
    xp = syn.random_intensities(w.batch, w.heads, L.p, seed=64, device="cuda")
    xc = syn.random_intensities(w.batch, w.heads, L.p, seed=65, device="cuda")
    P.update_online_mask(gt, rp, ci, hist, xp, xc)
    nre = P.map_rel_error(hist, gt).cpu().numpy()
    ref = O.reconstruct_history(gt.double().cpu().numpy(), h0, masks, masked_renorm=False)
    for h in range(w.heads):
        want = O.reconstruction_nre(ref[0, h], gt.double().cpu().numpy()[0, h])
        assert nre[0, h] == pytest.approx(want, rel=1e-12)
        assert 0 < nre[0, h] < math.inf


def test_map_rel_error_full_size(M):
    """Hunyuan 720p maps (n = 929, 24 heads) in the launch configuration the analysis script times."""
    w = syn.HUNYUAN
    L = olayout(w)
    P = M.Plan(w)
    A = syn.random_stats(w.batch, w.heads, L.n, seed=71, device="cuda")
    B = syn.random_stats(w.batch, w.heads, L.n, seed=72, device="cuda")
    out = P.map_rel_error(A, B).cpu().numpy()
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    for h in (0, 11, w.heads - 1):
        assert out[0, h] == pytest.approx(O.rel_frobenius(An[0, h], Bn[0, h]), rel=1e-12)
