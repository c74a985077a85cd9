"""App. C FLOP table (tests/golden/appc_flops.json) pins the FLOP-counting
convention used by bench.py: the paper counts 2*N^2*H*d per full attention (one multiply-add per
QK^T and PV term), bench.py counts 4*D*|I_i||I_j| FLOPs per selected block (2 FLOPs per MAC)."""
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
G = json.load(open(os.path.join(HERE, "golden", "appc_flops.json")))


def test_full_attention_and_overhead_identities():
    N, H, d = G["N"], G["H"], G["d"]
    assert round(2 * N * N * H * d / 1e12, 4) == G["full_attention_tflop"]
    assert round(N * N * H / 1e12, 4) == G["convert_to_sparsity_tflop"]
    p = 3 * G["n_blocks"] - 1 + G["frames"]
    assert round(p ** 3 / 3 / 1e12, 4) == G["solve_kernel_tflop"]                    # P:1300, one factorisation
    # "50% mask -> 74%": exactly dense QK^T + half of PV (reading Z25)
    assert abs(G["topk200_50pct_mask_tflop"] / G["full_attention_tflop"] - 0.75) < 1e-4


def test_bench_flop_count_convention():
    from bench import attn_flops
    n, N, blk, D, H = 4, 256, 64, 64, 2
    rp = np.tile(np.arange(n + 1) * n, (1, H, 1)).astype(np.int64)
    ci = np.tile(np.tile(np.arange(n), n), (1, H, 1)).astype(np.int64)
    assert attn_flops(rp, ci, N, blk, D) == 2 * (2 * N * N * H * D)   # all-ones CSR = twice the paper's MAC count
