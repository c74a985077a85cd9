"""ctypes binding of libmoddit.so (include/moddit.h).  Argument marshalling only.

The library is mandatory: importing this module raises if libmoddit.so is missing or does not
export the declared symbols -- there is no CPU or PyTorch fallback anywhere in the package.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MODDIT_LIB_OVERRIDE") or os.path.join(_HERE, "libmoddit.so")   # override: A/B experiments only

MOD_OK, MOD_ERR_USAGE, MOD_ERR_INPUT, MOD_ERR_NUMERICAL, MOD_ERR_CUDA, MOD_ERR_UNSUPPORTED = range(6)
STATUS_NAMES = {0: "MOD_OK", 1: "MOD_ERR_USAGE", 2: "MOD_ERR_INPUT", 3: "MOD_ERR_NUMERICAL", 4: "MOD_ERR_CUDA",
                5: "MOD_ERR_UNSUPPORTED"}
MOD_SELECT_TOPK, MOD_SELECT_THRESHOLD, MOD_SELECT_TOPMASS = 0, 1, 2
MOD_STAT_POOLED = 0
MOD_ATTN_DEFAULT, MOD_ATTN_SPLITKV, MOD_ATTN_PAIR, MOD_ATTN_WIDE = range(4)
ATTN_KERNELS = {"default": MOD_ATTN_DEFAULT, "splitkv": MOD_ATTN_SPLITKV, "pair": MOD_ATTN_PAIR, "wide": MOD_ATTN_WIDE}


class ModLayout(C.Structure):
    _fields_ = [("batch", C.c_int32), ("heads", C.c_int32), ("head_dim", C.c_int32),
                ("prefix_tokens", C.c_int32), ("frames", C.c_int32), ("height", C.c_int32),
                ("width", C.c_int32), ("block", C.c_int32)]


class ModConfig(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("tau_e", C.c_float), ("top_k", C.c_int32),
                ("select_mode", C.c_int32), ("select_param", C.c_float), ("stat_mode", C.c_int32),
                ("masked_renorm", C.c_int32), ("diag_guard", C.c_int32), ("softmax_scale", C.c_float),
                ("attn_kernel", C.c_int32)]


class ModSelection(C.Structure):
    _fields_ = [("select_mode", C.c_int32), ("top_k", C.c_int32), ("select_param", C.c_float)]


class ModditError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


P = C.c_void_p
I32 = C.c_int32

# name -> (restype, argtypes); must match include/moddit.h
SIGNATURES = {
    "mod_plan_create": (I32, [C.POINTER(ModLayout), C.POINTER(ModConfig), C.c_int, C.POINTER(P)]),
    "mod_plan_destroy": (None, [P]),
    "mod_plan_workspace_bytes": (C.c_size_t, [P]),
    "mod_plan_num_blocks": (I32, [P]),
    "mod_plan_num_patterns": (I32, [P]),
    "mod_plan_frame_blocks": (I32, [P, C.POINTER(I32)]),
    "mod_plan_diagnostics": (I32, [P, C.POINTER(C.c_double), C.POINTER(I32)]),
    "mod_plan_gram_inverse": (P, [P]),
    "mod_plan_gram_inverse_ld": (I32, [P]),
    "mod_plan_solver": (I32, [P]),
    "mod_plan_create_ms": (C.c_double, [P]),
    "mod_last_error": (C.c_char_p, []),
    "mod_version": (C.c_char_p, []),
    "mod_attn_kernel_name": (C.c_char_p, [P]),
    "mod_collect_block_stats": (I32, [P, P, P, P, P, P]),
    "mod_fit_mixture": (I32, [P, P, P, P, P, P]),
    "mod_keep_frames": (I32, [P, P, P, P, P]),
    "mod_predict_block_mask": (I32, [P, P, P, I32, I32, I32, P, C.POINTER(ModSelection), P, P, P, P]),
    "mod_update_online_mask": (I32, [P, P, P, P, P, P, P, P, P]),
    "mod_block_sparse_attn_fwd": (I32, [P, P, P, P, P, P, P, P, P, P]),
    "mod_fill_dense_mask": (I32, [P, P, P, P]),
    "mod_collect_exact_sparsity": (I32, [P, P, P, P, P, P, C.c_float, P, P, P]),
    "mod_quant_buffer_bytes": (C.c_size_t, [P]),
    "mod_quant_buffer_layout": (I32, [P, C.POINTER(C.c_size_t)]),
    "mod_quantize_qkv": (I32, [P, P, P, P, P, P]),
    "mod_block_sparse_attn_fwd_q8": (I32, [P, P, P, P, P, P, P, P]),
    "mod_map_rel_error": (I32, [P, P, P, P, P, P]),
    "mod_linearity_nre": (I32, [P, P, P, I32, I32, P, C.POINTER(I32), I32, P, P]),
    "mod_last_launch_count": (I32, []),
    "mod_ulysses_seq_pack": (I32, [P, P, I32, I32, I32, I32, I32, P]),
    "mod_ulysses_seq_unpack": (I32, [P, P, I32, I32, I32, I32, I32, P]),
    "mod_ulysses_head_pack": (I32, [P, P, I32, I32, I32, I32, I32, P]),
    "mod_ulysses_head_unpack": (I32, [P, P, I32, I32, I32, I32, I32, P]),
    "mod_ulysses_seq_pack_heads": (I32, [P, P, I32, I32, I32, I32, I32, I32, I32, P]),
    "mod_ulysses_head_unpack_heads": (I32, [P, P, I32, I32, I32, I32, I32, I32, I32, P]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libmoddit.so not built at {LIB_PATH}; run `python -m paper_2601_11641_b200.build` "
                          f"(or __graft_entry__.build()).  There is no fallback implementation.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)          # AttributeError = missing export: fail loudly
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    m = lib.mod_last_error()
    return m.decode() if m else ""


def check(status: int):
    if status != MOD_OK:
        raise ModditError(status, last_error())
