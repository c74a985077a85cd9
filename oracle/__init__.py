"""MOD-DiT oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 CPU implementation (numpy/scipy) of the hot path
of arxiv 2601.11641 ("MOD-DiT"), written from PAPER.md.  Every function cites the passage
it follows (``P:<line>`` = /root/reference/PAPER.md line, ``§`` = section, Eq./Alg./App.).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product package
``paper_2601_11641_b200`` never imports it and shares no code with it; the only thing both
sides share is the seeded input generator in ``synthetic/`` (no method arithmetic).

Readings of ambiguous passages are the SURVEY.md 8(c) "Z" readings, restated in DESIGN.md.
Parity pins live in ``tests/test_oracle_*.py``.  Functions without a pin independent of
themselves are marked "parity unpinned" below and in DESIGN.md:
  * ``pooled_block_stats``: no paper anchor (north-star construct); pinned by identities
    (block mean of token scores, rows sum to 1, closed form for constant blocks).
"""
from .layout import Layout, make_layout  # noqa: F401
from .stats import (pooled_block_stats, exact_sparsity, exact_sparsity_masked, exact_sparsity_masked_rows, sparsity_from_map,  # noqa: F401
                    informativeness_from_sparsity)  # noqa: F401
from .fit import (basis_C, basis_D, basis_E, design_matrix, gram_closed_form, gram_materialized,  # noqa: F401
                  rhs, rhs_materialized, solve_normal, fit_mixture, nae, reconstruct_from_x)
from .predict import (keep_frames, extrapolate, pattern_keys, select_patterns, block_mask,  # noqa: F401
                      mask_to_csr, csr_to_mask, predict_block_mask, SELECT_TOPK, SELECT_THRESHOLD,
                      SELECT_TOPMASS)
from .attention import masked_attention, masked_attention_rows, dense_attention  # noqa: F401
from .update import reconstruct_history, update_online_mask  # noqa: F401
from .schedule import OracleSchedule  # noqa: F401
from .analysis import rel_frobenius, der, reconstruction_nre, linearity_nre  # noqa: F401
from .quant import (round_e4m3, quantize_int8_blocks, quantize_e4m3_channels, dequantized_qkv,  # noqa: F401
                    quantized_attention_rows)
