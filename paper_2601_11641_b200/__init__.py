"""B200-native (sm_100a) MOD-DiT hot path (arxiv 2601.11641).

The product is ``libmoddit.so`` (C ABI, ``include/moddit.h``); this package is its thin Python
binding (``Plan``), the Algorithm-1 driver (``schedule``) and the head-parallel / Ulysses
helpers (``parallel``).  Importing it requires the built library -- there is no fallback.
"""
from ._lib import (MOD_SELECT_THRESHOLD, MOD_SELECT_TOPK, MOD_SELECT_TOPMASS, ModditError,  # noqa: F401
                   LIB_PATH, lib)
from .plan import LayoutSpec, Plan, last_launch_count  # noqa: F401

__version__ = lib.mod_version().decode()
