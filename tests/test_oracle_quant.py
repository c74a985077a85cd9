"""Pins for the oracle's quantized-attention path (reading Z30) -- no GPU.

The e4m3 rounding is pinned to torch's float8_e4m3fn cast (a library routine) and to hand-checked
values; the INT8 block quantization to closed forms; the attention to the exact path when the
inputs are already representable."""
import numpy as np
import pytest
import torch

import oracle as O


def test_round_e4m3_hand_values():
    cases = {1.0: 1.0, 0.0625: 0.0625, 3.14: 3.25, 3.1: 3.0, 447.0: 448.0, 1000.0: 448.0, -1000.0: -448.0,
             2.0 ** -9: 2.0 ** -9, 2.0 ** -10: 0.0, 1.0625: 1.0, 1.1875: 1.25, 0.0: 0.0, -17.0: -16.0}
    for x, want in cases.items():
        assert O.round_e4m3(np.float32(x)) == want, x
    # ties to even: 1.0625 lies halfway between 1.0 (mantissa 000) and 1.125 (001) -> 1.0;
    # 1.1875 halfway between 1.125 (001) and 1.25 (010) -> 1.25


def test_round_e4m3_matches_torch_float8():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000) * s for s in (1e-3, 0.05, 1, 30, 200)]).astype(np.float32)
    x = x[np.abs(x) <= 440]
    ref = torch.from_numpy(x).to(torch.float8_e4m3fn).to(torch.float64).numpy()
    assert np.array_equal(O.round_e4m3(x), ref)


def test_int8_block_quantization_closed_forms():
    L = O.make_layout(1, 1, 64, 0, 2, 8, 8, 64)          # N = 128, two blocks of 64 tokens
    rng = np.random.default_rng(1)
    X = rng.standard_normal((L.N, 64)).astype(np.float32)
    X[64:] = 0.0                                          # second block all zero
    X[5, 7] = 4.0                                         # block 0 absmax
    codes, scales = O.quantize_int8_blocks(X, L)
    assert scales[0] == np.float32(4.0) / np.float32(127.0) and scales[1] == 0.0
    assert codes[5, 7] == 127 and np.all(codes[64:] == 0)
    assert np.all(np.abs(codes) <= 127)
    # dequantization error is at most half a code step (plus fp32 rounding of the scale)
    err = np.abs(codes[:64].astype(np.float64) * np.float64(scales[0]) - X[:64])
    assert err.max() <= 0.5 * float(scales[0]) * (1 + 1e-6)


def test_e4m3_channel_quantization_closed_forms():
    rng = np.random.default_rng(2)
    V = rng.standard_normal((100, 8)).astype(np.float32)
    V[:, 3] = 0.0
    vals, scales = O.quantize_e4m3_channels(V)
    assert scales[3] == 0.0 and np.all(vals[:, 3] == 0)
    amax = np.abs(V).max(0)
    for d in (0, 1, 2):
        i = int(np.argmax(np.abs(V[:, d])))
        assert abs(vals[i, d]) == 448.0                       # the channel max maps to the e4m3 max
        assert scales[d] == np.float32(amax[d]) / np.float32(448.0)
    assert np.max(np.abs(vals)) <= 448.0


def test_quantized_attention_is_exact_on_representable_inputs():
    """If Q and K are integer multiples of absmax/127 and V of absmax_d/448 with e4m3 mantissas,
    quantization is the identity and the quantized attention equals the exact one."""
    L = O.make_layout(1, 1, 64, 0, 2, 8, 8, 64)
    rng = np.random.default_rng(3)
    qc = rng.integers(-127, 128, size=(L.N, 64)).astype(np.float32)
    kc = rng.integers(-127, 128, size=(L.N, 64)).astype(np.float32)
    qc[0, 0] = kc[0, 0] = qc[64, 0] = kc[64, 0] = 127.0      # each block reaches +127
    Q = (qc / np.float32(127.0)) * np.float32(1.5)           # block absmax 1.5 -> scale 1.5/127
    K = (kc / np.float32(127.0)) * np.float32(2.0)
    V = O.round_e4m3(rng.standard_normal((L.N, 64)).astype(np.float32) * 50).astype(np.float32)
    V[0, :] = 448.0                                           # channel absmax 448 -> scale 1
    mask = np.ones((L.n, L.n), dtype=bool)
    Qh, Kh, Vh, _ = O.dequantized_qkv(Q, K, V, L)
    assert np.allclose(Qh, Q, rtol=1e-6, atol=0) and np.allclose(Kh, K, rtol=1e-6, atol=0)
    assert np.array_equal(Vh, V.astype(np.float64))
    outs, _ = O.quantized_attention_rows(Q, K, V, mask, L, [0, 1])
    ref, _ = O.masked_attention_rows(Q.astype(np.float64)[None, None], K.astype(np.float64)[None, None],
                                     V.astype(np.float64)[None, None], mask, L, 0, 0, [0, 1])
    for a, b in zip(outs, ref):
        assert np.allclose(a, b, rtol=1e-5, atol=1e-5)
