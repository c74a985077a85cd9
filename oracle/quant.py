"""Oracle: quantized block-sparse attention -- TEST INFRASTRUCTURE ONLY.

The paper's sparse stage runs SageAttention ("SageAttention ... to reduce computational
overhead"), whose precision PAPER.md never states.  Reading Z30 fixes what this build's
quantized path computes, Sage-style:
  * Q and K: symmetric INT8 per 128-token block and head,  s = absmax / 127,  code = rint(x * (127 / absmax))
    in fp32 (round half to even), clipped to [-127, 127]; an all-zero block has s = 0 and codes 0;
  * V: FP8 e4m3 per channel (over all tokens) and head,  s_d = absmax_d / 448,  code = RN_e4m3(v * (448 / absmax_d))
    in fp32, saturating at +-448;
  * attention (Eq. 1) over the block mask with the dequantized Q^ = code*s, K^, V^.
The GPU additionally rounds the probabilities P to e4m3 before the PV product; that rounding is not
reproduced here (the parity bar in DESIGN.md covers it).  Integer decisions (the codes) are taken in
fp32 on both sides, as the kernel takes them, so they compare bit-exactly.
"""
from __future__ import annotations

import numpy as np

from .attention import masked_attention_rows
from .layout import Layout

E4M3_MAX = 448.0


def round_e4m3(y: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest e4m3 value (ties to even), saturating at +-448.
    e4m3: 1 sign, 4 exponent (bias 7), 3 mantissa bits; normal |y| >= 2^-6, subnormal step 2^-9."""
    y = np.asarray(y, dtype=np.float64)
    a = np.abs(y)
    e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    e = np.maximum(e, -6.0)                    # subnormals share the 2^-6 binade's quantum
    q = np.exp2(e - 3.0)                       # spacing of representable values in the binade
    r = np.rint(a / q) * q                     # np.rint: round half to even
    r = np.minimum(r, E4M3_MAX)
    return (np.sign(y) * r).astype(np.float64)


def quantize_int8_blocks(X: np.ndarray, L: Layout):
    """Per-(head, block) symmetric INT8 of one head's [N, D] tensor -> (codes int8 [N, D], scales fp32 [n])."""
    X = np.asarray(X, dtype=np.float32)
    codes = np.zeros(X.shape, dtype=np.int8)
    scales = np.zeros(L.n, dtype=np.float32)
    for i in range(L.n):
        lo, hi = L.block_range(i)
        blk = X[lo:hi]
        amax = np.float32(np.max(np.abs(blk))) if blk.size else np.float32(0)
        if amax > 0:
            inv = np.float32(127.0) / amax                      # fp32 division, as the kernel
            c = np.rint(blk * inv)                              # fp32 product, round half to even
            codes[lo:hi] = np.clip(c, -127, 127).astype(np.int8)
            scales[i] = amax / np.float32(127.0)
    return codes, scales


def quantize_e4m3_channels(V: np.ndarray):
    """Per-(head, channel) FP8 e4m3 of one head's [N, D] tensor -> (e4m3 values as fp64 [N, D], scales fp32 [D])."""
    V = np.asarray(V, dtype=np.float32)
    amax = np.max(np.abs(V), axis=0).astype(np.float32)
    inv = np.where(amax > 0, np.float32(E4M3_MAX) / np.where(amax > 0, amax, 1), 0).astype(np.float32)
    vals = round_e4m3((V * inv[None, :]).astype(np.float32))
    scales = (amax / np.float32(E4M3_MAX)).astype(np.float32)
    return vals, scales


def dequantized_qkv(Q: np.ndarray, K: np.ndarray, V: np.ndarray, L: Layout):
    """One head: the Q^, K^, V^ (fp64) the quantized path attends over, plus the raw codes/scales."""
    qc, qs = quantize_int8_blocks(Q, L)
    kc, ks = quantize_int8_blocks(K, L)
    vv, vs = quantize_e4m3_channels(V)
    blk = np.arange(L.N) // L.block
    Qh = qc.astype(np.float64) * qs.astype(np.float64)[blk][:, None]
    Kh = kc.astype(np.float64) * ks.astype(np.float64)[blk][:, None]
    Vh = vv * vs.astype(np.float64)[None, :]
    return Qh, Kh, Vh, (qc, qs, kc, ks, vv, vs)


def quantized_attention_rows(Q, K, V, mask: np.ndarray, L: Layout, qblocks, scale: float | None = None):
    """Eq. 1 over one head's block mask for the query blocks ``qblocks``, on the dequantized tensors
    (Q, K, V: that head's [N, D] arrays) -> (list of O blocks, list of lse blocks)."""
    Qh, Kh, Vh, _ = dequantized_qkv(Q, K, V, L)
    return masked_attention_rows(Qh[None, None], Kh[None, None], Vh[None, None], mask, L, 0, 0, qblocks, scale)
