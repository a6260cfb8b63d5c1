"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct FP64 CPU implementation of what the hot path
of Stiller, "Robust Multigrid for Cartesian Interior Penalty DG Formulations of
the Poisson Equation in 3D" (arXiv 1612.04796) computes.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import or execute anything under `oracle/`.  The product path
(`paper_1612_04796_b200`) never imports it and shares no code with it: the
only common module is `workloads/` (parameters + seeded random numbers).

Citations are `PAPER.md:<line>` (section / equation / algorithm) of
/root/reference/PAPER.md, or SPEC.md:<line>.

Two modes:
  * O-dense (`oracle.dense`): the global IP-DG matrix assembled explicitly from
    the 3D bilinear form (Eq. 4) with scipy.sparse; every Schwarz subdomain
    solved by dense LU of the principal submatrix A_ss = R_s A R_s^T (Eq. 9);
    coarse pseudo-inverse by pinned sparse LU (Alg. 1 l.295).
  * O-mf (`oracle.mf`): matrix-free equivalent (Eq. 7 Kronecker form from an
    independently assembled 1D IP matrix, fast diagonalisation with
    eigenpairs computed by mpmath at 40 digits).  Validated against O-dense on
    small grids; used for full-size parity and the timed CPU baseline.

Parity status of each function is listed in DESIGN.md §Oracle.  Functions
that no test pins against the paper or mathematics say "parity unpinned".
The only such item is the exact quintic of the hat weight beyond its stated
shape (oracle.overlap.hat_weight; reading R6).
"""
