"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the MOD-DiT method (no pooling, no fitting, no masks,
no attention).  It only draws random tensors with the shapes and structure of the
attention inputs named in BASELINE.json ``configs`` (recipe: DESIGN.md "Input recipe",
SURVEY.md 8(d)).  Both sides -- ``oracle/`` and the CUDA path -- receive the very same
bytes from here; neither imports the other.

Token order inside a head is ``[prefix | frame-major, y, x]``.
"""
from __future__ import annotations

import dataclasses
import math

import torch

SEED_BASE = 20260117


@dataclasses.dataclass(frozen=True)
class Workload:
    """Shape of one attention call: Q, K, V in [B, H, N, D] bf16, N = prefix + F*Hh*Ww."""
    name: str
    batch: int
    heads: int
    head_dim: int
    prefix_tokens: int
    frames: int
    height: int
    width: int
    block: int

    @property
    def tokens(self) -> int:
        return self.prefix_tokens + self.frames * self.height * self.width

    @property
    def num_blocks(self) -> int:
        return -(-self.tokens // self.block)

    def with_heads(self, heads: int) -> "Workload":
        return dataclasses.replace(self, heads=heads)

    def as_dict(self) -> dict:
        d = dataclasses.asdict(self)
        d["tokens"] = self.tokens
        return d


# BASELINE.json "configs" (entries 0..3); config 4 is Hunyuan sequence-sharded over 8 GPUs.
TINY = Workload("tiny", 1, 2, 64, 0, 4, 8, 8, 64)
COGVIDEOX = Workload("cogvideox-5b", 1, 48, 64, 226, 13, 30, 45, 128)
WAN = Workload("wan2.1-14b-720p", 1, 40, 128, 0, 21, 45, 80, 128)
HUNYUAN = Workload("hunyuanvideo-720p", 1, 24, 128, 0, 33, 45, 80, 128)
CONFIGS = {w.name: w for w in (TINY, COGVIDEOX, WAN, HUNYUAN)}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def family_r(w: Workload, seed: int = SEED_BASE, device="cpu"):
    """Family R (parity): Q, K, V i.i.d. N(0, 1), rounded to bf16."""
    shape = (w.batch, w.heads, w.tokens, w.head_dim)
    out = []
    for t in range(3):
        g = _gen(seed + t, device)
        out.append(torch.randn(shape, generator=g, device=device, dtype=torch.float32).to(torch.bfloat16))
    return tuple(out)


def family_s(w: Workload, seed: int = SEED_BASE, device="cpu", sigma: float = 0.5,
             kappa: float = 1.0, n_random_sinks: int = 2, step: int = 0, head_offset: int = 0,
             total_heads: int | None = None, drift: float = 0.0, steps_total: int = 50):
    """Family S (structured): planted intra-frame, inter-frame and global-column structure.

    Q = a_h*phi(y,x) + b_h*psi(f) + c_h*g_h + sigma*eps
    K = a_h*phi(y,x) + b_h*psi(f) + kappa*[block in sinks_h]*g_h + sigma*eps
    phi: smooth random-Fourier spatial features; psi(f), g_h, eps ~ N(0, I);
    (a_h, b_h, c_h) ~ Dirichlet(1,1,1)*scale per head; sinks = block 0 plus
    ``n_random_sinks`` seeded random blocks per head; V ~ N(0, 1).  Each tensor is
    rescaled to unit per-element variance, then rounded to bf16.
    ``step`` re-draws only the noise eps (emulates consecutive denoising steps with the same
    structure).  ``head_offset``/``total_heads`` generate the heads [head_offset, head_offset+H) of a
    ``total_heads``-head problem (head-parallel ranks draw exactly the bytes a single GPU would).
    ``drift`` > 0 makes the pattern strengths evolve over the denoising steps (the piecewise-smooth
    intensity trajectories of PAPER.md §4.3): with tau = step / steps_total, the spatial,
    temporal and sink weights of head h become a_h*(1 + d1*tau + d2*tau^2), etc., with per-head
    (d1, d2) ~ U(-drift, drift) drawn from their own generator (drift = 0 leaves every byte unchanged).
    """
    B, H, N, D = w.batch, w.heads, w.tokens, w.head_dim
    HT = total_heads or H
    g = _gen(seed, "cpu")
    # small per-head / per-frame parameters are drawn on the CPU (cheap, device independent)
    dirich = torch.distributions.Dirichlet(torch.ones(3))
    torch.manual_seed(seed)  # Dirichlet uses the global generator; seed it for determinism
    abc = dirich.sample((HT,)) * 2.0                                    # [HT, 3]
    half = D // 2
    om = torch.rand((half, 2), generator=g) * 0.5 * (16.0 / max(w.height, w.width))
    ph0 = torch.rand((half,), generator=g) * 2 * math.pi
    psi = torch.randn((w.frames, D), generator=g)                        # [F, D]
    gh = torch.randn((HT, D), generator=g)                               # [HT, D]
    n = w.num_blocks
    sink_mask = torch.zeros((HT, n), dtype=torch.bool)
    sink_mask[:, 0] = True
    for h in range(HT):
        idx = torch.randint(0, n, (n_random_sinks,), generator=g)
        sink_mask[h, idx] = True
    # spatial features for the video tokens, [HW, D]
    yy, xx = torch.meshgrid(torch.arange(w.height, dtype=torch.float32),
                            torch.arange(w.width, dtype=torch.float32), indexing="ij")
    arg = yy.reshape(-1, 1) * om[:, 0] + xx.reshape(-1, 1) * om[:, 1] + ph0       # [HW, half]
    phi = torch.cat([torch.cos(arg), torch.sin(arg)], dim=1) * math.sqrt(2.0)     # [HW, D]
    HW = w.height * w.width
    dev = torch.device(device)
    phi_t = torch.zeros((N, D))
    psi_t = torch.zeros((N, D))
    phi_t[w.prefix_tokens:] = phi.repeat(w.frames, 1)
    psi_t[w.prefix_tokens:] = psi.repeat_interleave(HW, dim=0)
    tok_block = torch.arange(N) // w.block
    if drift:
        gd = _gen(seed + 5, "cpu")
        dco = (torch.rand((HT, 3, 2), generator=gd, dtype=torch.float64) * 2 - 1) * drift
        tau = step / float(steps_total)
        fac = 1.0 + dco[..., 0] * tau + dco[..., 1] * tau * tau                 # [HT, 3]: a, b, kappa
    else:
        fac = torch.ones((HT, 3), dtype=torch.float64)
    phi_t, psi_t = phi_t.to(dev), psi_t.to(dev)
    q = torch.empty((B, H, N, D), dtype=torch.bfloat16, device=dev)
    k = torch.empty_like(q)
    for hl in range(H):
        h = head_offset + hl
        gen_dev = _gen(seed + 1 + 1000 * step + 7919 * h, dev)
        a, b, c = (float(x) for x in abc[h])
        a, b = a * float(fac[h, 0]), b * float(fac[h, 1])
        kap = kappa * float(fac[h, 2])
        ghh = gh[h].to(dev)
        sinks_tok = sink_mask[h][tok_block].to(dev).float().unsqueeze(1)          # [N, 1]
        for bb in range(B):
            eq = torch.randn((N, D), generator=gen_dev, device=dev)
            ek = torch.randn((N, D), generator=gen_dev, device=dev)
            qh = a * phi_t + b * psi_t + c * ghh + sigma * eq
            kh = a * phi_t + b * psi_t + kap * sinks_tok * ghh + sigma * ek
            if w.prefix_tokens:
                qh[: w.prefix_tokens] = torch.randn((w.prefix_tokens, D), generator=gen_dev, device=dev)
                kh[: w.prefix_tokens] = torch.randn((w.prefix_tokens, D), generator=gen_dev, device=dev)
            q[bb, hl] = (qh / qh.std()).to(torch.bfloat16)
            k[bb, hl] = (kh / kh.std()).to(torch.bfloat16)
    v = torch.empty_like(q)
    for hl in range(H):
        gv = _gen(seed + 2 + 7919 * (head_offset + hl), dev)
        v[:, hl] = torch.randn((B, N, D), generator=gv, device=dev, dtype=torch.float32).to(torch.bfloat16)
    return q, k, v


def family_s_heads(w: Workload, heads, **kw):
    """Family S for an arbitrary list of heads of ``w`` (e.g. a rank's LPT or Ulysses-chunk heads): the
    heads are generated one at a time (``head_offset`` = h, ``total_heads`` = w.heads), so every head's
    bytes equal those of the full tensor and at most one head is live beyond the output."""
    outs = [family_s(w.with_heads(1), head_offset=int(h), total_heads=w.heads, **kw) for h in heads]
    return tuple(torch.cat([o[i] for o in outs], dim=1) for i in range(3))


def family_s_seq_shard(w: Workload, t0: int, t1: int, **kw):
    """Tokens [t0, t1) of every head of Family S, in the sequence-sharded activation layout [B, t1-t0, H, D]
    (the input of a Ulysses rank).  Generated head by head, so a rank never holds the full tensors."""
    B, H, D = w.batch, w.heads, w.head_dim
    dev = kw.get("device", "cpu")
    outs = tuple(torch.empty((B, t1 - t0, H, D), dtype=torch.bfloat16, device=dev) for _ in range(3))
    for h in range(H):
        qkv = family_s(w.with_heads(1), head_offset=h, total_heads=H, **kw)
        for dst, src in zip(outs, qkv):
            dst[:, :, h] = src[:, 0, t0:t1]
    return outs


def random_stats(B: int, H: int, n: int, seed: int = SEED_BASE, device="cpu") -> torch.Tensor:
    """Row-stochastic fp32 block-statistic maps [B,H,n,n] (positive, rows sum to ~1)."""
    g = _gen(seed, device)
    x = torch.rand((B, H, n, n), generator=g, device=device, dtype=torch.float64) ** 4
    return (x / x.sum(-1, keepdim=True)).to(torch.float32)


def random_intensities(B: int, H: int, p: int, seed: int = SEED_BASE, device="cpu") -> torch.Tensor:
    g = _gen(seed, device)
    return torch.randn((B, H, p), generator=g, device=device, dtype=torch.float64)
