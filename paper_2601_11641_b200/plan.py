"""Python face of the C ABI: ``Plan`` wraps one ``mod_plan`` and the six compute calls.

PyTorch is used only for device memory (output / workspace tensors) and the current CUDA stream;
every step of the hot path runs in libmoddit.so's kernels.  Calls are asynchronous on
``torch.cuda.current_stream()`` exactly like the C functions.
"""
from __future__ import annotations

import ctypes as C
import dataclasses

import torch

from . import _lib
from ._lib import ModConfig, ModLayout, ModSelection, check, lib


@dataclasses.dataclass(frozen=True)
class LayoutSpec:
    batch: int
    heads: int
    head_dim: int
    prefix_tokens: int
    frames: int
    height: int
    width: int
    block: int = 128

    @property
    def tokens(self) -> int:
        return self.prefix_tokens + self.frames * self.height * self.width

    @classmethod
    def from_any(cls, w) -> "LayoutSpec":
        if isinstance(w, LayoutSpec):
            return w
        if isinstance(w, dict):
            return cls(**{f.name: w[f.name] for f in dataclasses.fields(cls)})
        return cls(**{f.name: getattr(w, f.name) for f in dataclasses.fields(cls)})


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _stream(device=None):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _on_device(fn):
    """Run a compute call with the plan's device current, so that its launches go to that device's
    current stream (the C library launches on the stream it is given, with the caller's current device)."""
    import functools

    @functools.wraps(fn)
    def wrapped(self, *a, **kw):
        with torch.cuda.device(self.device):
            return fn(self, *a, **kw)
    return wrapped


class Plan:
    """Per-layout constants (block/frame ranges, deflated Gram inverse) + the compute calls."""

    def __init__(self, layout, *, top_k: int = 1, lam: float = 1e-8, tau_e: float = 0.0,
                 select_mode: int = _lib.MOD_SELECT_TOPK, select_param: float = 0.0,
                 masked_renorm: bool = True, diag_guard: bool = True, softmax_scale: float = 0.0,
                 attn_kernel: str = "default", device: int | None = None):
        self.spec = LayoutSpec.from_any(layout)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._cl = ModLayout(*(getattr(self.spec, f) for f in
                               ("batch", "heads", "head_dim", "prefix_tokens", "frames", "height", "width",
                                "block")))
        if attn_kernel not in _lib.ATTN_KERNELS:
            raise ValueError(f"attn_kernel={attn_kernel!r} must be one of {sorted(_lib.ATTN_KERNELS)}")
        self._cc = ModConfig(lam, tau_e, top_k, select_mode, select_param, _lib.MOD_STAT_POOLED,
                             int(masked_renorm), int(diag_guard), softmax_scale, _lib.ATTN_KERNELS[attn_kernel])
        self.config = dict(lam=lam, tau_e=tau_e, top_k=top_k, select_mode=select_mode, select_param=select_param,
                           masked_renorm=masked_renorm, diag_guard=diag_guard, softmax_scale=softmax_scale,
                           attn_kernel=attn_kernel)
        h = C.c_void_p()
        check(lib.mod_plan_create(C.byref(self._cl), C.byref(self._cc), self.device, C.byref(h)))
        self._h = h
        self.n = lib.mod_plan_num_blocks(h)
        self.p = lib.mod_plan_num_patterns(h)
        fb = (C.c_int32 * (2 * self.spec.frames))()
        check(lib.mod_plan_frame_blocks(h, fb))
        self.frame_blocks = [(fb[2 * r], fb[2 * r + 1]) for r in range(self.spec.frames)]
        mp, nd = C.c_double(), C.c_int32()
        check(lib.mod_plan_diagnostics(h, C.byref(mp), C.byref(nd)))
        self.min_pivot, self.null_dim = mp.value, nd.value
        # App. B P:1251-1270 solver chain step that produced the Gram inverse, and the plan build time
        self.solver = ("cholesky", "lu", "pinv")[lib.mod_plan_solver(h)]
        self.create_ms = lib.mod_plan_create_ms(h)
        self.ws_bytes = lib.mod_plan_workspace_bytes(h)
        self._ws = {}        # one workspace per CUDA stream (moddit.h: concurrent calls need their own)
        # softmax scale s: 1/sqrt(head_dim) unless given
        self.scale = softmax_scale if softmax_scale > 0 else 1.0 / float(self.spec.head_dim) ** 0.5

    # ------------------------------------------------------------------ plumbing
    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:   # module globals may already be torn down at interpreter exit
            lib.mod_plan_destroy(h)
            self._h = None

    def attn_kernel_name(self) -> str:
        """The K4 kernel instantiation this plan launches (from the library)."""
        return lib.mod_attn_kernel_name(self._h).decode()

    @property
    def handle(self):
        return self._h

    @property
    def BH(self) -> int:
        return self.spec.batch * self.spec.heads

    @property
    def N(self) -> int:
        return self.spec.tokens

    def workspace(self, stream=None) -> torch.Tensor:
        """The workspace of ``stream`` (default: the current stream of the plan's device).  Calls on
        different streams get different workspaces, so one Plan can serve several streams at once."""
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        ws = self._ws.get(st.cuda_stream)
        if ws is None:
            ws = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device=f"cuda:{self.device}")
            self._ws[st.cuda_stream] = ws
        return ws

    def _check(self, name, t, dtype, shape, optional=False):
        """Argument check the C side cannot do on device pointers: dtype, shape, device, contiguity."""
        if t is None:
            if optional:
                return
            raise ValueError(f"{name} is required")
        if t.dtype != dtype or tuple(t.shape) != tuple(shape) or not t.is_cuda or t.device.index != self.device \
                or not t.is_contiguous():
            raise ValueError(f"{name}: expected contiguous {dtype} tensor of shape {tuple(shape)} on cuda:{self.device}, "
                             f"got {t.dtype} {tuple(t.shape)} on {t.device}"
                             f"{'' if t.is_contiguous() else ' (non-contiguous)'}")

    def _check_stats(self, name, t):
        self._check(name, t, torch.float32, (self.spec.batch, self.spec.heads, self.n, self.n))

    def _check_x(self, name, t):
        self._check(name, t, torch.float64, (self.spec.batch, self.spec.heads, self.p))

    def _check_csr(self, rp, ci):
        B, H, n = self.spec.batch, self.spec.heads, self.n
        self._check("row_ptr", rp, torch.int32, (B, H, n + 1))
        self._check("col_idx", ci, torch.int32, (B, H, n * n))

    def _dev(self):
        return torch.device(f"cuda:{self.device}")

    def _check_qkv(self, *ts):
        B, H, N, D = self.spec.batch, self.spec.heads, self.N, self.spec.head_dim
        for t in ts:
            if t.shape != (B, H, N, D) or t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous() \
                    or t.device.index != self.device:
                raise ValueError(f"expected contiguous bf16 CUDA tensor of shape {(B, H, N, D)}, got "
                                 f"{tuple(t.shape)} {t.dtype} {t.device} (plan device cuda:{self.device})")

    def empty_stats(self) -> torch.Tensor:
        return torch.empty((self.spec.batch, self.spec.heads, self.n, self.n), dtype=torch.float32, device=self._dev())

    def empty_x(self) -> torch.Tensor:
        return torch.empty((self.spec.batch, self.spec.heads, self.p), dtype=torch.float64, device=self._dev())

    def empty_mask(self):
        B, H, n = self.spec.batch, self.spec.heads, self.n
        return (torch.empty((B, H, n + 1), dtype=torch.int32, device=self._dev()),
                torch.empty((B, H, n * n), dtype=torch.int32, device=self._dev()))

    # ------------------------------------------------------------------ compute calls
    @_on_device
    def collect_block_stats(self, q, k, out=None):
        self._check_qkv(q, k)
        out = self.empty_stats() if out is None else out
        self._check_stats("out", out)
        check(lib.mod_collect_block_stats(self._h, _ptr(q), _ptr(k), _ptr(out), _ptr(self.workspace()), _stream()))
        return out

    @_on_device
    def fit_mixture(self, stats, out=None, want_nae: bool = False):
        self._check_stats("stats", stats)
        out = self.empty_x() if out is None else out
        self._check_x("out", out)
        nae = torch.empty((self.spec.batch, self.spec.heads), dtype=torch.float32, device=self._dev()) if want_nae else None
        check(lib.mod_fit_mixture(self._h, _ptr(stats), _ptr(out), _ptr(nae), _ptr(self.workspace()), _stream()))
        return (out, nae) if want_nae else out

    @_on_device
    def keep_frames(self, x_a, x_b):
        self._check_x("x_a", x_a)
        self._check_x("x_b", x_b)
        keep = torch.empty((self.spec.batch, self.spec.heads, self.spec.frames), dtype=torch.uint8, device=self._dev())
        check(lib.mod_keep_frames(self._h, _ptr(x_a), _ptr(x_b), _ptr(keep), _stream()))
        return keep

    @_on_device
    def predict_block_mask(self, x_prev, x_curr, t_prev: int, t_curr: int, t: int, keep=None, *,
                           select_mode: int | None = None, top_k: int | None = None,
                           select_param: float | None = None, out=None):
        self._check_x("x_prev", x_prev)
        self._check_x("x_curr", x_curr)
        self._check("keep", keep, torch.uint8, (self.spec.batch, self.spec.heads, self.spec.frames), optional=True)
        rp, ci = self.empty_mask() if out is None else out
        self._check_csr(rp, ci)
        sel = None
        if select_mode is not None or top_k is not None or select_param is not None:
            sel = ModSelection(self.config["select_mode"] if select_mode is None else select_mode,
                               self.config["top_k"] if top_k is None else top_k,
                               self.config["select_param"] if select_param is None else select_param)
        check(lib.mod_predict_block_mask(self._h, _ptr(x_prev), _ptr(x_curr), t_prev, t_curr, t, _ptr(keep),
                                         C.byref(sel) if sel is not None else None, _ptr(rp), _ptr(ci),
                                         _ptr(self.workspace()), _stream()))
        return rp, ci

    @_on_device
    def update_online_mask(self, stats_fresh, row_ptr, col_idx, stats_hist, x_prev, x_curr):
        self._check_stats("stats_fresh", stats_fresh)
        self._check_stats("stats_hist", stats_hist)
        self._check_csr(row_ptr, col_idx)
        self._check_x("x_prev", x_prev)
        self._check_x("x_curr", x_curr)
        check(lib.mod_update_online_mask(self._h, _ptr(stats_fresh), _ptr(row_ptr), _ptr(col_idx), _ptr(stats_hist),
                                         _ptr(x_prev), _ptr(x_curr), _ptr(self.workspace()), _stream()))

    @_on_device
    def block_sparse_attn_fwd(self, q, k, v, row_ptr, col_idx, out=None, lse=None, want_lse: bool = True):
        self._check_qkv(q, k, v)
        self._check_csr(row_ptr, col_idx)
        out = torch.empty_like(q) if out is None else out
        self._check_qkv(out)
        if lse is None and want_lse:
            lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=q.device)
        self._check("lse", lse, torch.float32, tuple(q.shape[:-1]), optional=True)
        check(lib.mod_block_sparse_attn_fwd(self._h, _ptr(q), _ptr(k), _ptr(v), _ptr(row_ptr), _ptr(col_idx),
                                            _ptr(out), _ptr(lse), _ptr(self.workspace()), _stream()))
        return out, lse

    @_on_device
    def collect_exact_sparsity(self, q, k, lse, row_ptr, col_idx, eta: float = 1e-4, out=None):
        """U = -S of Eq. 2 for the listed blocks (unlisted entries of ``out`` untouched)."""
        self._check_qkv(q, k)
        self._check("lse", lse, torch.float32, tuple(q.shape[:-1]))
        self._check_csr(row_ptr, col_idx)
        out = self.empty_stats().fill_(float("nan")) if out is None else out
        self._check_stats("out", out)
        check(lib.mod_collect_exact_sparsity(self._h, _ptr(q), _ptr(k), _ptr(lse), _ptr(row_ptr), _ptr(col_idx),
                                             eta, _ptr(out), _ptr(self.workspace()), _stream()))
        return out

    # ------------------------------------------------------------------ quantized attention (f2)
    @_on_device
    def quant_buffer(self) -> torch.Tensor:
        """Caller-owned buffer for the quantized operands (layout: include/moddit.h, reading Z30)."""
        nbytes = lib.mod_quant_buffer_bytes(self._h)
        if nbytes == 0:
            check(lib.mod_quant_buffer_layout(self._h, (C.c_size_t * 6)()))   # raises with the reason
        return torch.empty(nbytes, dtype=torch.uint8, device=self._dev())

    def quant_views(self, qbuf: torch.Tensor) -> dict:
        """Typed views of a quantized-operand buffer: q8, k8 int8 [B,H,N,D]; vt8 uint8 (e4m3 bits)
        [B,H,D,Np]; q_scale, k_scale fp32 [B,H,n]; v_scale fp32 [B,H,D]."""
        off = (C.c_size_t * 6)()
        check(lib.mod_quant_buffer_layout(self._h, off))
        B, H, N, D, n = self.spec.batch, self.spec.heads, self.N, self.spec.head_dim, self.n
        Np = (N + 15) // 16 * 16

        def view(o, count, dtype, shape):
            return qbuf[o:o + count * torch.tensor([], dtype=dtype).element_size()].view(dtype).view(shape)
        return {"q8": view(off[0], B * H * N * D, torch.int8, (B, H, N, D)),
                "k8": view(off[1], B * H * N * D, torch.int8, (B, H, N, D)),
                "vt8": view(off[2], B * H * D * Np, torch.uint8, (B, H, D, Np)),
                "q_scale": view(off[3], B * H * n, torch.float32, (B, H, n)),
                "k_scale": view(off[4], B * H * n, torch.float32, (B, H, n)),
                "v_scale": view(off[5], B * H * D, torch.float32, (B, H, D))}

    @_on_device
    def quantize_qkv(self, q, k, v, out=None) -> torch.Tensor:
        self._check_qkv(q, k, v)
        qbuf = self.quant_buffer() if out is None else out
        check(lib.mod_quantize_qkv(self._h, _ptr(q), _ptr(k), _ptr(v), _ptr(qbuf), _stream()))
        return qbuf

    @_on_device
    def block_sparse_attn_fwd_q8(self, qbuf, row_ptr, col_idx, out=None, lse=None, want_lse: bool = True):
        B, H, N, D = self.spec.batch, self.spec.heads, self.N, self.spec.head_dim
        o = torch.empty((B, H, N, D), dtype=torch.bfloat16, device=self._dev()) if out is None else out
        self._check_qkv(o)
        self._check_csr(row_ptr, col_idx)
        if lse is None and want_lse:
            lse = torch.empty((B, H, N), dtype=torch.float32, device=self._dev())
        self._check("lse", lse, torch.float32, (B, H, N), optional=True)
        check(lib.mod_block_sparse_attn_fwd_q8(self._h, _ptr(qbuf), _ptr(row_ptr), _ptr(col_idx), _ptr(o), _ptr(lse),
                                               _ptr(self.workspace()), _stream()))
        return o, lse

    # ------------------------------------------------------------------ analysis metrics (f3)
    @_on_device
    def map_rel_error(self, a, b, out=None):
        """||a - b||_F / ||b||_F per head (DER; reconstruction NRE) -> fp64 [B, H]."""
        for t in (a, b):
            if t.dtype != torch.float32 or tuple(t.shape) != (self.spec.batch, self.spec.heads, self.n, self.n) \
                    or not t.is_contiguous():
                raise ValueError(f"maps must be contiguous fp32 {[self.spec.batch, self.spec.heads, self.n, self.n]}")
        out = torch.empty((self.spec.batch, self.spec.heads), dtype=torch.float64, device=self._dev()) \
            if out is None else out
        check(lib.mod_map_rel_error(self._h, _ptr(a), _ptr(b), _ptr(out), _ptr(self.workspace()), _stream()))
        return out

    @_on_device
    def linearity_nre(self, x_prev, x_curr, t_prev: int, t_curr: int, x_traj, t_steps):
        """App. A linearity NRE of the C/D intensities over the steps ``t_steps`` -> fp64
        [B, H, 3n-1]; ``x_traj`` is fp64 [S, B, H, p] (the fits at those steps)."""
        S = len(t_steps)
        if tuple(x_traj.shape) != (S, self.spec.batch, self.spec.heads, self.p) or x_traj.dtype != torch.float64 \
                or not x_traj.is_contiguous():
            raise ValueError(f"x_traj must be contiguous fp64 {[S, self.spec.batch, self.spec.heads, self.p]}")
        ts = (C.c_int32 * max(S, 1))(*[int(t) for t in t_steps])
        out = torch.empty((self.spec.batch, self.spec.heads, 3 * self.n - 1), dtype=torch.float64, device=self._dev())
        check(lib.mod_linearity_nre(self._h, _ptr(x_prev), _ptr(x_curr), t_prev, t_curr, _ptr(x_traj), ts, S,
                                    _ptr(out), _stream()))
        return out

    @_on_device
    def dense_mask(self, out=None):
        rp, ci = self.empty_mask() if out is None else out
        self._check_csr(rp, ci)
        check(lib.mod_fill_dense_mask(self._h, _ptr(rp), _ptr(ci), _stream()))
        return rp, ci


def last_launch_count() -> int:
    return lib.mod_last_launch_count()
