"""fp64 CPU oracle for the randomized Krylov f(A)b method (arXiv 2212.12758).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import, call
or execute anything under ``oracle/``.  The product path
(``paper_2212_12758_b200``) never imports it and shares no code with it.

Plain, slow, obviously correct: each function follows the paper's algorithm
step by step, in the paper's order and notation, and cites the passage it
implements as ``PAPER.md l.<line>`` (section / algorithm / equation).  Readings
where the paper is silent or garbled are the G-n entries of SURVEY.md §8c-2,
restated in DESIGN.md "Readings".

Modules
  rng     SplitMix64 counter hash: SRHT signs and sampled rows (G-10)
  srht    Walsh-Hadamard transform and the SRHT Theta, and
          the one-entry definition used for full-size spot checks
  krylov  Alg 2 truncated orthogonalization, Arnoldi (Eq. 2), Alg 1
          sketched Gram-Schmidt (l.76-100), Alg 2 with whitening (l.106, l.395)
  lsq     Householder QR, triangular solve, LSQR, Blendenpik, sketch-and-solve
  matfun  f(C) e_1 for f in {exp, sqrt, invsqrt, poly}
  fab     drivers: Alg 4, Alg 5, sketch-and-solve (Remark 2), sFOM Eq. (9),
          Arnoldi FOM Eq. (4), Alg 3 (l.187-197), the whitened variants,
          sign(A) b by (A^2)^{-1/2} (A b) (l.406), dense reference

Parity pins: tests/test_oracle_*.py.  Nothing here is "parity unpinned"
except the numerical values of unconverged approximants, which have no
external truth.
"""
from . import rng, srht, krylov, lsq, matfun, fab  # noqa: F401
