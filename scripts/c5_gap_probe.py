"""Measure the GPU-vs-oracle iterate and residual gaps of plain V(1,1) cycles on c5 (AR 48):
the data behind tests/tolerances.py's anisotropic bars.  Diagnostic."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1612_04796_b200 import DG
from workloads import get_config, uniform_zero_mean
from oracle.mf import MFHierarchy
from oracle import mg

for ne in (3, None):
    c = get_config("c5", ne)
    g = DG(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    H = MFHierarchy(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    f = uniform_zero_mean(c.ndofs, 0)
    fg = torch.from_numpy(f).cuda()
    ug = torch.zeros_like(fg)
    u = np.zeros_like(f)
    for k in range(3):
        g.pmg_vcycle(ug, fg)
        u = mg.vcycle(H, u, f)
        un = ug.cpu().numpy()
        gap = np.max(np.abs(un - u)) / np.max(np.abs(u))
        rg = np.max(np.abs(H.apply(H.L, un - u))) / np.max(np.abs(f))
        print("c5 ne=%s cycle %d  iterate gap %.3e  residual gap %.3e  |r|/|r0| %.3e" % (
            ne, k + 1, gap, rg, mg.residual_norm(H, u, f) / np.linalg.norm(f)), flush=True)
