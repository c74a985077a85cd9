"""Shared helpers of the GPU parity tests (conversions only; no method arithmetic)."""
from __future__ import annotations

import numpy as np
import torch

import oracle as O

FIELDS = ("batch", "heads", "head_dim", "prefix_tokens", "frames", "height", "width", "block")


def olayout(w) -> "O.Layout":
    return O.make_layout(*[getattr(w, f) for f in FIELDS])


def masks_to_csr(masks: np.ndarray, device="cuda"):
    """Per-head bool masks [B,H,n,n] -> (row_ptr [B,H,n+1], col_idx [B,H,n*n]) int32 CUDA tensors."""
    B, H, n, _ = masks.shape
    rp = np.zeros((B, H, n + 1), dtype=np.int32)
    ci = np.full((B, H, n * n), -1, dtype=np.int32)
    for b in range(B):
        for h in range(H):
            r, c = O.mask_to_csr(masks[b, h])
            rp[b, h] = r
            ci[b, h, : len(c)] = c
    return torch.from_numpy(rp).to(device), torch.from_numpy(ci).to(device)


def csr_to_masks(rp: torch.Tensor, ci: torch.Tensor, n: int) -> np.ndarray:
    rp = rp.cpu().numpy()
    ci = ci.cpu().numpy()
    B, H = rp.shape[:2]
    out = np.zeros((B, H, n, n), dtype=bool)
    for b in range(B):
        for h in range(H):
            out[b, h] = O.csr_to_mask(rp[b, h], ci[b, h], n)
    return out


def csr_rows_sorted_unique(rp: torch.Tensor, ci: torch.Tensor, n: int) -> bool:
    rp = rp.cpu().numpy()
    ci = ci.cpu().numpy()
    for b in range(rp.shape[0]):
        for h in range(rp.shape[1]):
            r = rp[b, h]
            if r[0] != 0 or np.any(np.diff(r) < 0):
                return False
            for i in range(n):
                row = ci[b, h, r[i]:r[i + 1]]
                if len(row) and (np.any(np.diff(row) <= 0) or row.min() < 0 or row.max() >= n):
                    return False
    return True


def null_vector_c_d(n: int, p: int) -> np.ndarray:
    """Unit vector (1_C, -1_D, 0_E)/norm: sum_k C_k = J = sum_k D_k (App. B)."""
    v = np.zeros(p)
    v[: 2 * n - 1] = 1.0
    v[2 * n - 1: 3 * n - 1] = -1.0
    return v / np.linalg.norm(v)
