"""Parity bars of the GPU-vs-oracle tests, each with the arithmetic it comes from.

TOL (1e-11): BASELINE.json north_star — relative max-norm error of the operator apply, the
    smoother, the transfers, the coarse solve and one V-cycle's iterate.
TOL_ANISO (5e-10), TOL_ANISO_RES (1e-10): c5 and other element aspect ratios ~48 only.  There
    the subdomain operators have kappa(A_ss) ~ 1e6 and the two EXACT FP64 oracles of the
    subdomain solve — dense LU of A_ss (oracle.dense) and fast diagonalisation (oracle.mf) —
    already disagree on c5's element shape (3^3 elements, P = 8 GL, MaxRelative(0.08)+floor 1):
    iterate 8.0e-11 after one V(1,1) cycle and 1.24e-10 after two; residual of the difference
    2.0e-11 of ||f||.  tests/test_oracle_floor.py re-measures that floor on every CPU run and
    asserts these bars stay >= 4x (iterate) / 5x (residual) above it and that TOL itself is below
    it (so the exception is needed, not a convenience).  The GPU measured 7.6e-11 / 1.18e-10
    (iterate) and 1.9e-11 / 2.1e-11 (residual) on the same grid (scripts/c5_gap_probe.py).
"""
TOL = 1e-11
TOL_ANISO = 5e-10
TOL_ANISO_RES = 1e-10
