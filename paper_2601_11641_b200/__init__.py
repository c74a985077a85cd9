"""B200-native (sm_100a) MOD-DiT hot path (arxiv 2601.11641).

The product is ``libmoddit.so`` (C ABI, ``include/moddit.h``); this package is its thin Python
binding (``Plan``), the Algorithm-1 driver (``schedule``) and the head-parallel / Ulysses
helpers (``parallel``).  Using it requires the built library -- there is no fallback; the library is
loaded on first use (so that ``python -m paper_2601_11641_b200.build`` works on a fresh checkout).
"""
_LIB_NAMES = ("MOD_SELECT_THRESHOLD", "MOD_SELECT_TOPK", "MOD_SELECT_TOPMASS", "ModditError", "LIB_PATH", "lib")
_PLAN_NAMES = ("LayoutSpec", "Plan", "last_launch_count")


def __getattr__(name):
    if name in _LIB_NAMES:
        from . import _lib
        return getattr(_lib, name)
    if name in _PLAN_NAMES:
        from . import plan
        return getattr(plan, name)
    if name == "__version__":
        from . import _lib
        return _lib.lib.mod_version().decode()
    raise AttributeError(name)


__all__ = list(_LIB_NAMES + _PLAN_NAMES)
