"""Pins for oracle O5-O8 (keep, extrapolate, select, mask, CSR) -- no GPU.

Pinned by SPEC.md worked examples, brute-force sorting and
set-union enumeration written independently here.
"""
import itertools

import numpy as np
import pytest

import oracle as O


def test_extrapolate_spec_examples():
    assert O.extrapolate(0.5, 0.5, 12, 22, 30) == 0.5
    assert O.extrapolate(0.4, 0.6, 22, 32, 37) == pytest.approx(0.7, abs=1e-15)
    with pytest.raises(ValueError):
        O.extrapolate(0.1, 0.2, 5, 5, 7)


def test_extrapolate_exact_on_linear_and_affine():
    a, b = 0.37, -1.25
    for (tp, tc, t) in [(11, 12, 13), (12, 22, 29), (22, 32, 42)]:
        xp, xc = a * tp + b, a * tc + b
        assert O.extrapolate(xp, xc, tp, tc, t) == pytest.approx(a * t + b, abs=1e-12)
        # affine invariance
        s, o = 3.0, 0.25
        assert O.extrapolate(s * xp + o, s * xc + o, tp, tc, t) == pytest.approx(
            s * O.extrapolate(xp, xc, tp, tc, t) + o, abs=1e-12)


def test_keep_frames_spec():
    L = O.make_layout(1, 1, 64, 0, 1, 1, 8, 8)   # n=1, p=3, one frame: e at index 2
    ka = lambda ea, eb, tau: int(O.keep_frames([0, 0, ea], [0, 0, eb], L, tau)[0])
    assert ka(0.9, 0.8, 0.5) == 1
    assert ka(0.5, 0.9, 0.5) == 0       # S:292 strict
    assert ka(0.2, 0.9, 0.5) == 0


def _brute_topk(keys, K):
    order = sorted(range(len(keys)), key=lambda i: (-keys[i], i))
    return set(order[:K])


def test_select_topk_descending_ties():
    n = 2                                   # pool of 5: C(-1,0,1), D(0,1)
    keys = np.array([0.1, 0.9, 0.2, 0.9, 0.3])
    assert set(np.nonzero(O.select_patterns(keys, n, O.SELECT_TOPK, 2))[0]) == {1, 3}
    assert set(np.nonzero(O.select_patterns(keys, n, O.SELECT_TOPK, 1))[0]) == {1}   # tie -> lower id
    assert O.select_patterns(keys, n, O.SELECT_TOPK, 99).all()                       # clip
    eq = np.zeros(5)
    assert set(np.nonzero(O.select_patterns(eq, n, O.SELECT_TOPK, 3))[0]) == {0, 1, 2}


def test_select_topk_brute_force_and_monotone():
    rng = np.random.default_rng(0)
    n = 6
    keys = np.round(rng.standard_normal(3 * n - 1), 1)     # many ties
    prev = set()
    for K in range(1, 3 * n):
        s = set(np.nonzero(O.select_patterns(keys, n, O.SELECT_TOPK, K))[0])
        assert s == _brute_topk(list(keys), K)
        assert prev <= s                                    # monotone in K
        prev = s


def test_select_threshold_and_topmass():
    rng = np.random.default_rng(1)
    n = 5
    keys = rng.standard_normal(3 * n - 1)
    th = O.select_patterns(keys, n, O.SELECT_THRESHOLD, param=0.3)
    assert np.array_equal(th, keys > 0.3)
    supp = [n - abs(k - (n - 1)) for k in range(2 * n - 1)] + [n] * n
    order = sorted(range(3 * n - 1), key=lambda i: (-keys[i], i))
    mass = [max(keys[i], 0.0) * supp[i] for i in order]
    total = sum(mass)
    for rho in (0.1, 0.5, 0.9, 1.0):
        sel = O.select_patterns(keys, n, O.SELECT_TOPMASS, param=rho)
        acc, Lp = 0.0, None
        for t, m in enumerate(mass):
            acc += m
            if acc >= rho * total:
                Lp = t + 1
                break
        assert set(np.nonzero(sel)[0]) == set(order[:Lp])


def _enum_mask(sel, keep, L, guard):
    n = L.n
    pas = set()
    for k in range(2 * n - 1):
        if sel[k]:
            d = k - (n - 1)
            pas |= {(i, i + d) for i in range(n) if 0 <= i + d < n}
    for k in range(n):
        if sel[2 * n - 1 + k]:
            pas |= {(i, k) for i in range(n)}
    for r in range(L.frames):
        if keep[r]:
            a, b = L.frame_blocks(r)
            pas |= set(itertools.product(range(a, b + 1), repeat=2))
    if guard:
        pas |= {(i, i) for i in range(n)}
    pl = L.prefix_last_block
    pas |= {(i, j) for i in range(n) for j in range(n) if i <= pl or j <= pl}
    return pas


@pytest.mark.parametrize("P0,F,HW,b", [(0, 2, 8, 4), (0, 4, 64, 64), (5, 3, 20, 8), (30, 4, 33, 16)])
def test_block_mask_is_union_of_supports(P0, F, HW, b):
    L = O.make_layout(1, 1, 64, P0, F, 1, HW, b)
    rng = np.random.default_rng(F + HW)
    for trial in range(5):
        sel = rng.random(3 * L.n - 1) < 0.3
        keep = (rng.random(F) < 0.5).astype(np.uint8)
        guard = bool(trial % 2)
        m = O.block_mask(sel, keep, L, guard)
        got = set(zip(*np.nonzero(m)))
        assert got == _enum_mask(sel, keep, L, guard)      # S:370 set-union oracle
        rp, ci = O.mask_to_csr(m)
        assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == len(got)
        for i in range(L.n):
            row = ci[rp[i]:rp[i + 1]]
            assert np.all(np.diff(row) > 0)                 # sorted, unique
        assert np.array_equal(O.csr_to_mask(rp, ci, L.n), m)


def test_mask_spec_examples():
    L = O.make_layout(1, 1, 64, 0, 1, 1, 8, 4)      # n = 2, one frame covering the grid
    sel = np.zeros(5, dtype=bool)
    sel[1] = True                                   # main diagonal only
    m = O.block_mask(sel, np.array([0]), L, diag_guard=False)
    assert set(zip(*np.nonzero(m))) == {(0, 0), (1, 1)}
    m = O.block_mask(np.zeros(5, dtype=bool), np.array([1]), L, diag_guard=False)
    assert m.all()
    L4 = O.make_layout(1, 1, 64, 0, 2, 1, 8, 4)     # n = 4
    m = np.zeros((4, 4), dtype=bool)
    m[0, 0] = m[1, 2] = m[3, 1] = True
    assert 1 - m.sum() / 16 == 0.8125                            # S:366 sparsity ratio
    assert L4.n == 4


def test_exact_polarity_is_the_papers_ascending_topk_on_fit_of_S():
    """Reading Z3 with U = -S (EXACT statistic): the descending Top-K on fit(U) must be exactly the
    paper's literal rule, "Top-K ... in ascending order" of the intensities fitted to S (§5.3),
    ties by pattern id.  (U = 1 - S would add the per-family offset fit(J) -- C: n/(3n-1),
    D: (2n-1)/(3n-1), App. Z.5 -- and select different patterns, which this test also shows.)"""
    L = O.make_layout(1, 1, 8, 0, 3, 4, 4, 4)                # n = 12, F = 3
    n = L.n
    rng = np.random.default_rng(21)
    differs = 0
    for trial in range(6):
        S = rng.random((1, 1, n, n))
        xS = O.fit_mixture(S, L)[0, 0]
        xU = O.fit_mixture(O.informativeness_from_sparsity(S), L)[0, 0]
        assert np.array_equal(xU, -xS)                        # the solve is odd in its right-hand side
        pool = 3 * n - 1
        for K in (1, 5, 8, 20):
            literal = np.zeros(pool, dtype=bool)
            literal[np.lexsort((np.arange(pool), xS[:pool]))[:K]] = True   # ascending on fit(S), ties by id
            assert np.array_equal(O.select_patterns(O.pattern_keys(xU, L), n, O.SELECT_TOPK, K), literal)
            x1 = O.fit_mixture(1.0 - S, L)[0, 0]
            differs += not np.array_equal(O.select_patterns(O.pattern_keys(x1, L), n, O.SELECT_TOPK, K), literal)
    assert differs > 0
