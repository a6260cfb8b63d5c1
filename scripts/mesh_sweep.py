#!/usr/bin/env python
"""NEXT row f2 (Fig. 5): average convergence rate of GLL MG with
delta_O = 0.08 Delta x versus the number of elements N_e = k^3 on the 2pi-periodic cube, for
P = 4, 8, 16, 32; paper protocol as in table1_sweep.py.  The paper: mesh independent for
N_e >~ 12^3 at P <= 16, still improving beyond 16^3 at P = 32; rho ~ 6.3e-3 (P=16) and
1.6e-3 (P=32)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from workloads.configs import OverlapSpec
from scripts.table1_sweep import run_case

GRIDS = {4: [4, 8, 12, 16, 24, 32], 8: [4, 8, 12, 16, 24], 16: [4, 8, 12, 16], 32: [4, 8, 12]}


def main():
    for P, ks in GRIDS.items():
        for k in ks:
            res = run_case("GLL", "MG", OverlapSpec(1, 0.08, 0), P, k)
            print("P=%2d N_e=%2d^3  DOF=%9d  rho=%.3e  -lg rho=%.2f  cycles=%d" % (
                P, k, res["dofs"], res["rho"], res["lg"], res["cycles"]), flush=True)


if __name__ == "__main__":
    main()
