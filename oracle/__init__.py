"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation of what the GBS hot path
computes (§2.1 Eq. (1) and the Richardson combination, lines 85-115,
186-225; §3.7 Eqs. (5)-(6), lines 403-425), written from the paper and pinned
to things other than itself (tests/test_oracle_*.py, tests/golden/).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import, call, link or
execute anything under ``oracle/``.  The product package
``paper_1907_11771_b200`` never imports it, and the two share no code: they
meet only at the seeded inputs of ``gbs_inputs`` and at fp64 weights/H values
each side derives independently from exact rationals.

Modules
  gbs_oracle.c  fp64 stepping (FE, LF, averaging, weighted sum) on the MOL FD
                right-hand sides and the 1-D spectral derivative (a plain O(N^2)
                DFT); built into _build/liboracle_gbs.so
  c_oracle      ctypes wrapper of the C library
  weights       exact-rational extrapolation weights (Eq. 3, 5, 6)
  stability     exact GBS stability polynomials, R(iy) scan, ISB, rho, H rule
  fd            exact centered FD coefficients (Taylor conditions) and symbols
  fourier       closed-form per-Fourier-mode solution of the linear configs
  exact         exact-rational (Fraction) brute-force stepping on tiny grids

Parity status: every function above is pinned;
none is "parity unpinned" except the choice of ICs and of the all-nonzero
parity weight set, which the paper does not fix.  The
Appendix-B optimised free weights (gbs_inputs/optimized_schemes.json, weight
set "opt8") are inputs written by the product's optimiser; the oracle checks
them independently (exact order 8, its own ISB scan) and computes their
dependent weights itself.
"""
