"""POBK oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the POBK hot path computes
(arXiv 2401.00672, PAPER.md; readings in SURVEY.md §8(c) and DESIGN.md §3).  It exists to
prove the CUDA path correct and to time a CPU baseline; it is NOT a fallback.

Who may import / call / link / execute anything under oracle/:
  * tests/                      (pins and parity tests)
  * __graft_entry__.smoke()     (one small parity check on cuda:0)
  * bench.py                    (the cpu_baseline leg and `--impl reference` only)
The product package paper_2401_00672_b200/ never imports it, and the two share no code:
no kernels, headers, helpers, tables, constant generators, pre- or post-processing.  The
only shared module is workloads/ (seeded input generators, no method arithmetic).

Layout:
  oracle/c/pobk_oracle.c  plain C: RCM (O2-O3), first-fit (O5-O6), the row-by-row sweep
                          Eq 1.2 (O7), RSE/RELRES (O8), the solve loop
  oracle/core.py          Python wrappers + O1 canonicalisation, O4 permutation,
                          O6 schedule, O9 back-permutation, and pure-Python/NumPy
                          restatements used on small cases

Parity status per function is listed in DESIGN.md §3 ("what pins each part").  The sweep
counts on the synthetic configs are "parity unpinned" by the paper (no paper values
exist for these inputs); they are pinned only oracle <-> GPU.
"""
from .core import *  # noqa: F401,F403
