"""ORACLE -- plain, slow, obviously-correct CPU implementation of the method.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product path (``paper_1806_10284_b200``) never imports, links or
executes anything here, and this package never imports the product path.
The two share no code; only ``synthetic/`` (seeded inputs, no method
arithmetic) serves both.

Modules (each function cites the PAPER.md passage it follows):
  lattice   §2.2-2.3  canonicalisation, angle snapping, eq. (transvec),
                      reciprocal lattice, reduced Bloch numbers
  curl      §3        Yee curl C by geometric quasi-periodic wrap; the
                      paper's explicit K1, K2/J2 and 4-category J3 forms;
                      B; dense GEP C*C e = lambda B e (plain definition)
  spectral  §4-5      closed-form eigenpairs of K1..K3, dense T, Lambda_q,
                      Pi0/Pi1/Pi2, Q, P, SVD, dense A_r (naive O(n^2) DFT)
  fftop     §5.3      matrix-free A_r via Algorithms 1-2 (numpy FFTs)
  eigsolve  §5.2, §6  inverse Lanczos + CG (paper's solver), block variant

Precision: float64 / complex128 throughout (PAPER.md L2398 tolerances imply
FP64).  Readings of garbled or ambiguous passages are listed in DESIGN.md
("Readings"); each is cited where it is used.

Parity status: every function is pinned by a ``-m "not gpu"`` test in
tests/test_oracle_*.py against something other than itself (worked
examples, closed forms, invariants, textbook DFT, brute force); none is
"parity unpinned".
"""
