"""One pass of every libmoddit kernel family on small layouts, for compute-sanitizer (memcheck, synccheck,
racecheck, initcheck): K1 statistics, K2a fit (+ NAE), keep, K2b predict (Top-K / threshold / top-mass),
K3 update, K4 attention (default, splitkv, pair; dense and sparse lists, empty rows, ragged tails),
f1 EXACT statistic, f2 quantize + quantized attention, f3 analysis metrics, the Ulysses relayouts.
  compute-sanitizer --tool memcheck python scripts/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthetic as syn  # noqa: E402
from paper_2601_11641_b200 import Plan  # noqa: E402
from paper_2601_11641_b200.parallel import KERNELS  # noqa: E402

SMALL_PREFIX = syn.Workload("small-prefix", 1, 2, 128, 40, 3, 20, 19, 128)   # ragged tail 28
COG_SMALL = syn.Workload("cog-small", 1, 2, 64, 226, 3, 30, 45, 128)         # D = 64, prefix, ragged 52
for w in (syn.TINY, SMALL_PREFIX, COG_SMALL):
    for kern in ("default", "splitkv", "pair"):
        P = Plan(w, top_k=4, tau_e=0.0, attn_kernel=kern)
        q1, k1, _ = syn.family_s(w, step=11, device="cuda")
        q, k, v = syn.family_s(w, step=12, device="cuda")
        W1, W2 = P.collect_block_stats(q1, k1), P.collect_block_stats(q, k)
        x1, (x2, nae) = P.fit_mixture(W1), P.fit_mixture(W2, want_nae=True)
        keep = P.keep_frames(x1, x2)
        for mode, par in ((0, None), (1, 0.0), (2, 0.5)):
            kw = {"top_k": 4} if mode == 0 else {"select_mode": mode, "select_param": par}
            rp, ci = P.predict_block_mask(x1, x2, 11, 12, 22, keep, **kw)
        rp, ci = P.predict_block_mask(x1, x2, 11, 12, 22, keep, top_k=4)
        o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
        rpd, cid = P.dense_mask()
        od, lsed = P.block_sparse_attn_fwd(q, k, v, rpd, cid)
        rpe = rp.clone()
        rpe[..., 1:] = rpe[..., :1]          # every row empty
        P.block_sparse_attn_fwd(q, k, v, rpe, ci)
        hist = W2.clone()
        P.update_online_mask(P.collect_block_stats(q, k), rp, ci, hist, x1, x2)
        if kern == "default":
            P.collect_exact_sparsity(q, k, lsed, rpd, cid, 1e-4)
            P.collect_exact_sparsity(q, k, lse, rp, ci, 1e-4)
            if w.head_dim == 128 and w.block == 128:
                qb = P.quant_buffer()
                P.quantize_qkv(q, k, v, out=qb)
                P.block_sparse_attn_fwd_q8(qb, rp, ci)
            P.map_rel_error(W1, W2)
    torch.cuda.synchronize()
B, N, H, D = 1, 8 * 150, 24, 128
x = torch.randn((B, N, H, D), device="cuda").to(torch.bfloat16)
for Pn in (1, 2, 4):
    s = KERNELS.seq_pack(x[:, : N // Pn].contiguous(), Pn)
    xh = KERNELS.seq_unpack(s)
    KERNELS.head_unpack(KERNELS.head_pack(xh, Pn))
    KERNELS.seq_pack_heads(x, 8, 8, Pn if 8 % Pn == 0 else 1)
torch.cuda.synchronize()
print("sanitize_run ok")
