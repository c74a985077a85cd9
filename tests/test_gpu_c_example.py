"""The plain-C consumer of the C ABI (examples/moddit_step.c) against the Python binding on the same
inputs: same kernels, same call sequence, so outputs must be bit-identical (the library is
deterministic, include/moddit.h)."""
import os
import subprocess

import numpy as np
import pytest
import torch

import synthetic as syn

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W = syn.Workload("c-example", 1, 3, 128, 40, 3, 20, 19, 128)   # N=1180, n=10, ragged tail 28


def test_c_example_matches_python_binding(tmp_path):
    from paper_2601_11641_b200 import Plan
    from paper_2601_11641_b200.build import build_examples
    exe = os.path.join(ROOT, "examples", "moddit_step")
    if not os.path.exists(exe):
        build_examples()
    q, k, v = syn.family_s(W, device="cuda")
    q1, k1, _ = syn.family_s(W, step=1, device="cuda")
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as f:
        for t in (q, k, v, q1, k1):
            f.write(t.view(torch.int16).cpu().numpy().tobytes())
    out = tmp_path / "out.bin"
    top_k = 5
    r = subprocess.run([exe, "1", "3", "128", "40", "3", "20", "19", "128", str(top_k), str(inp), str(out)],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    # the same step through the Python binding
    P = Plan(W, top_k=top_k)
    W1, W2 = P.collect_block_stats(q1, k1), P.collect_block_stats(q, k)
    xp, xc = P.fit_mixture(W1), P.fit_mixture(W2)
    keep = P.keep_frames(xp, xc)
    rp, ci = P.predict_block_mask(xp, xc, 11, 12, 13, keep)
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    P.update_online_mask(P.collect_block_stats(q, k), rp, ci, W2, xp, xc)
    torch.cuda.synchronize()
    buf = out.read_bytes()
    BH, N, n, p = 3, W.tokens, P.n, P.p
    off = 0
    o_c = np.frombuffer(buf, dtype=np.int16, count=BH * N * 128, offset=off)
    off += BH * N * 128 * 2
    lse_c = np.frombuffer(buf, dtype=np.float32, count=BH * N, offset=off)
    off += BH * N * 4
    rp_c = np.frombuffer(buf, dtype=np.int32, count=BH * (n + 1), offset=off)
    off += BH * (n + 1) * 4
    xc_c = np.frombuffer(buf, dtype=np.float64, count=BH * p, offset=off)
    assert np.array_equal(o_c, o.view(torch.int16).cpu().numpy().ravel())
    assert np.array_equal(lse_c, lse.cpu().numpy().ravel())
    assert np.array_equal(rp_c, rp.cpu().numpy().ravel())
    assert np.array_equal(xc_c, xc.cpu().numpy().ravel())
    assert "moddit_step ok" in r.stdout
