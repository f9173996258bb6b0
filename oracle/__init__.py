"""Plain float64 / complex128 CPU oracle for the QTT convolution hot path of
arXiv 2301.13339 (Alg. 1 TT-SVD, QTT-FFT contract, Alg. 2 QTT
convolution, Alg. 3 Full).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path
(`paper_2301_13339_b200/`, `include/`) may import, call or link this package.
Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl
reference` legs of `bench.py` use it.  It shares no code with the CUDA path:
the two meet only at the seeded input generators
(`paper_2301_13339_b200/synth.py`, which holds none of the method's
arithmetic).

Every function cites the PAPER.md passage it follows ("P:<line>") and, where
the paper is silent, the reading from SURVEY.md §8(c) it implements
("Q<n>" / "O<n>"); DESIGN.md §3 lists all readings.

Parity status:
  * tt_svd / rank_rule / full          — pinned (closed forms, paper ranks
                                          17/26/26, storage Tables 3/5,
                                          exact reconstruction, Lemma 1).
  * qfft / qifft / center / hadamard   — pinned (numpy.fft, closed-form DFTs,
                                          Parseval, per-stage invariant).
  * rank_rule_dropoff (modification 3) — pinned (rule cases, exact low rank,
                                          Table 1 I_delta, Example 2 exact).
  * rng.omega / qtt.rsvd_step          — pinned (N(0,1) statistics,
    (modification 2, TT-RSVD)            exactness on low rank, Eq.
                                          rsvd_error bound, fallback rule,
                                          Table 1 I_QTT_r).
  * round_full / conv_pipeline         — pinned at eps=0 by brute-force
                                          periodic convolution; with caps by
                                          the paper's Table 1 E2 band for
                                          Example 1.
"""

from .qtt import (axes_descriptor, to_qtt, from_qtt, rank_rule, rank_rule_dropoff, choose_rank, margin_log,
                  tt_svd, full, element, storage_count, ranks_of)
from .qfft import qfft, qifft, center, hadamard, round_full, round_local
from .conv import conv_pipeline
from . import rng

__all__ = [
    "axes_descriptor", "to_qtt", "from_qtt", "rank_rule", "rank_rule_dropoff", "choose_rank", "margin_log",
    "tt_svd", "full",
    "element", "storage_count", "ranks_of", "qfft", "qifft", "center",
    "hadamard", "round_full", "round_local", "conv_pipeline",
]
