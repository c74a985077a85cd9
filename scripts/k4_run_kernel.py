"""k4_run.py with the K4 schedule given by its mod_attn_kernel enum value (for variant libraries whose
schedules the current binding does not name).  python scripts/k4_run_kernel.py CONFIG ENUM [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synthetic as syn
import paper_2601_11641_b200 as M
from paper_2601_11641_b200 import _lib

_lib.ATTN_KERNELS.setdefault("k" + sys.argv[2], int(sys.argv[2]))
w = syn.CONFIGS[sys.argv[1]]
P = M.Plan(w, top_k=1, attn_kernel="k" + sys.argv[2])
q1, k1, _ = syn.family_s(w, step=11, device="cuda")
W1 = P.collect_block_stats(q1, k1)
del q1, k1
q, k, v = syn.family_s(w, step=12, device="cuda")
W2 = P.collect_block_stats(q, k)
x1, x2 = P.fit_mixture(W1), P.fit_mixture(W2)
K = {"cogvideox-5b": 12, "wan2.1-14b-720p": 96}.get(sys.argv[1], 164)
rp, ci = P.predict_block_mask(x1, x2, 11, 12, 22, P.keep_frames(x1, x2), top_k=K)
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
torch.cuda.synchronize()
print("ok", P.attn_kernel_name())
