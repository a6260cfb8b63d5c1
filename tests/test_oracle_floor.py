"""The FP64 floor of c5 (AR 48): two exact oracles of the same V(1,1) cycle — dense LU of every
restricted operator A_ss (Eq. 9) vs fast diagonalisation —
differ by rounding only, and this difference sets the anisotropic parity bars (tolerances.py)."""
import numpy as np

from workloads import get_config, uniform_zero_mean
from oracle.dense import DenseHierarchy
from oracle.mf import MFHierarchy
from oracle import mg
from tolerances import TOL, TOL_ANISO, TOL_ANISO_RES


def test_c5_two_exact_oracles_floor_sets_aniso_bars():
    c = get_config("c5", 3)                   # c5's element shape and levels, 3^3 elements
    Hd = DenseHierarchy(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    Hm = MFHierarchy(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    f = uniform_zero_mean(Hd.ndofs(Hd.L), 0)
    a = np.zeros_like(f)
    b = np.zeros_like(f)
    gaps, rgaps = [], []
    for _ in range(2):
        a = mg.vcycle(Hd, a, f)
        b = mg.vcycle(Hm, b, f)
        gaps.append(np.max(np.abs(a - b)) / np.max(np.abs(a)))
        rgaps.append(np.max(np.abs(Hm.apply(Hm.L, a - b))) / np.max(np.abs(f)))
    # the two exact solves agree to the conditioning-limited floor ...
    assert max(gaps) <= TOL_ANISO / 4, gaps
    assert max(rgaps) <= TOL_ANISO_RES / 4, rgaps
    # ... which lies above the isotropic bar: that is why c5 has its own bars
    assert max(gaps) > TOL, gaps
