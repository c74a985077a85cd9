"""O5-O8 -- keep-frames, linear prediction, pattern selection, block mask, CSR (oracle).

Test infrastructure only.
* keep (§5.3, Alg. 1; readings Z3, Z6, Z7): keep_r = min(e_r^(m-1), e_r^(m)) > tau_e.
* extrapolation (§5.2 Eq. 6, Eq. 7; Alg. 1): for the C and D
  parts only, x_hat = x_c + (x_c - x_p) / (t_c - t_p) * (t - t_c); E is never predicted.
  Evaluated in IEEE fp64 in exactly this order: d = x_c - x_p; s = d / (t_c - t_p);
  x_hat = x_c + s * (t - t_c)  (no fused multiply-add).
* selection (§5.3; reading Z3 polarity "informativeness", Z14 ties): the pool is the
  3n-1 patterns C_0..C_{2n-2}, D_0..D_{n-1} (ids 0..3n-2).  TOPK: sort by key descending, ties
  by pattern id ascending (C before D), take the first min(K, 3n-1).  THRESHOLD: key > theta.
  TOPMASS (BASELINE.json north_star "top-mass"): shortest prefix of the sorted list whose
  running sum of max(key,0)*|supp| (sequential fp64 sum in sorted order) reaches
  rho * (the full sum); |supp(C_k)| = n - |delta_k|, |supp(D_k)| = n.
* mask (§5.3, Alg. 1; readings Z15, Z17): pass(i,j) iff j-i = delta_k for a
  selected C_k, or j = k for a selected D_k, or (i,j) in [a_r,b_r]^2 for a kept frame r, or
  (diag_guard and i = j), or i or j is a prefix block.
* CSR: per row the ascending list of passing j (the "index list" of the north star).
"""
from __future__ import annotations

import numpy as np

from .layout import Layout

SELECT_TOPK, SELECT_THRESHOLD, SELECT_TOPMASS = 0, 1, 2


def keep_frames(x_a, x_b, L: Layout, tau_e: float = 0.0) -> np.ndarray:
    x_a = np.asarray(x_a, dtype=np.float64)
    x_b = np.asarray(x_b, dtype=np.float64)
    o = 3 * L.n - 1
    ea, eb = x_a[..., o:o + L.frames], x_b[..., o:o + L.frames]
    return (np.minimum(ea, eb) > tau_e).astype(np.uint8)


def extrapolate(x_prev, x_curr, t_prev: int, t_curr: int, t: int) -> np.ndarray:
    """Eq. 6/7 on the C and D entries (returns the 3n-1 predicted keys per head)."""
    x_prev = np.asarray(x_prev, dtype=np.float64)
    x_curr = np.asarray(x_curr, dtype=np.float64)
    if t_curr == t_prev:
        raise ValueError("t_prev == t_curr (zero denominator)")
    d = x_curr - x_prev
    s = d / np.float64(t_curr - t_prev)
    return x_curr + s * np.float64(t - t_curr)


def pattern_keys(x_hat, L: Layout) -> np.ndarray:
    return np.asarray(x_hat, dtype=np.float64)[..., : 3 * L.n - 1]


def _supp_sizes(n: int) -> np.ndarray:
    return np.array([n - abs(k - (n - 1)) for k in range(2 * n - 1)] + [n] * n, dtype=np.float64)


def select_patterns(keys: np.ndarray, n: int, mode: int = SELECT_TOPK, top_k: int = 1,
                    param: float = 0.0) -> np.ndarray:
    """Boolean selection over the 3n-1 pool for ONE head."""
    keys = np.asarray(keys, dtype=np.float64)
    P = 3 * n - 1
    assert keys.shape == (P,)
    sel = np.zeros(P, dtype=bool)
    if mode == SELECT_THRESHOLD:
        return keys > param
    # descending key, ascending id: lexsort sorts by last key first
    order = np.lexsort((np.arange(P), -keys))
    if mode == SELECT_TOPK:
        sel[order[: min(top_k, P)]] = True
        return sel
    if mode == SELECT_TOPMASS:
        mass = np.maximum(keys[order], 0.0) * _supp_sizes(n)[order]
        cum = np.zeros(P)
        acc = 0.0
        for t in range(P):              # sequential fp64 sum in sorted order
            acc = acc + mass[t]
            cum[t] = acc
        total = acc
        if not total > 0.0:
            return sel
        target = param * total
        L_ = int(np.argmax(cum >= target)) + 1 if np.any(cum >= target) else P
        sel[order[:L_]] = True
        return sel
    raise ValueError(f"bad select mode {mode}")


def block_mask(sel: np.ndarray, keep: np.ndarray, L: Layout, diag_guard: bool = True) -> np.ndarray:
    """n x n boolean pass mask for ONE head."""
    n = L.n
    mask = np.zeros((n, n), dtype=bool)
    for k in range(2 * n - 1):
        if sel[k]:
            mask |= basis_support_C(n, k)
    for k in range(n):
        if sel[2 * n - 1 + k]:
            mask[:, k] = True
    for r in range(L.frames):
        if keep[r]:
            a, b = L.frame_blocks(r)
            mask[a:b + 1, a:b + 1] = True
    if diag_guard:
        mask |= np.eye(n, dtype=bool)
    pl = L.prefix_last_block
    if pl >= 0:
        mask[: pl + 1, :] = True
        mask[:, : pl + 1] = True
    return mask


def basis_support_C(n: int, k: int) -> np.ndarray:
    d = k - (n - 1)
    m = np.zeros((n, n), dtype=bool)
    for i in range(n):
        if 0 <= i + d < n:
            m[i, i + d] = True
    return m


def mask_to_csr(mask: np.ndarray):
    """row_ptr [n+1], col_idx [nnz] (ascending per row) for ONE head."""
    n = mask.shape[0]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    cols = []
    for i in range(n):
        js = np.nonzero(mask[i])[0]
        cols.append(js)
        row_ptr[i + 1] = row_ptr[i] + len(js)
    col_idx = np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)
    return row_ptr, col_idx.astype(np.int64)


def csr_to_mask(row_ptr, col_idx, n: int) -> np.ndarray:
    m = np.zeros((n, n), dtype=bool)
    row_ptr = np.asarray(row_ptr)
    col_idx = np.asarray(col_idx)
    for i in range(n):
        m[i, col_idx[row_ptr[i]:row_ptr[i + 1]]] = True
    return m


def predict_block_mask(x_prev, x_curr, t_prev, t_curr, t, keep, L: Layout, mode=SELECT_TOPK,
                       top_k=1, param=0.0, diag_guard=True):
    """Per-head masks [B,H,n,n] from (x_prev, x_curr) (Alg. 1)."""
    x_hat = extrapolate(x_prev, x_curr, t_prev, t_curr, t)
    keys = pattern_keys(x_hat, L)
    lead = keys.shape[:-1]
    kf = keys.reshape(-1, keys.shape[-1])
    kp = np.asarray(keep).reshape(-1, L.frames)
    out = np.zeros((kf.shape[0], L.n, L.n), dtype=bool)
    for t_ in range(kf.shape[0]):
        sel = select_patterns(kf[t_], L.n, mode, top_k, param)
        out[t_] = block_mask(sel, kp[t_], L, diag_guard)
    return out.reshape(lead + (L.n, L.n))
