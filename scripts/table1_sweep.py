#!/usr/bin/env python
"""NEXT row f2: Table 1 sweep on the GPU.  14 cases (basis x solver x overlap)
x P = 4, 8, 16, 32 on N_e = (128/P)^3 elements of the 2pi-periodic cube, V(1,1), paper protocol:
random initial guess in [-1,1] (seeded), RHS = M (3 sin x sin y sin z) (the paper's own manufactured
solution is garbled), iterate until ||r_n||/||r_0|| <= 1e-10, rho = (r_n/r_0)^(1/n).
Writes profiles/<tag>_table1_gpu.json and prints a markdown table next to the paper's values."""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_1612_04796_b200 import DG
from workloads.configs import OverlapSpec
from workloads import uniform_vector

PAPER = {  # row: (basis, solver, overlap, [P=4, 8, 16, 32])
    1: ("GLL", "MG", OverlapSpec(0, 1, 0), [1.08, 0.89, 0.46, 0.24]),
    2: ("GLL", "MG-CG", OverlapSpec(0, 1, 0), [1.34, 1.21, 0.80, 0.52]),
    3: ("GLL", "MG", OverlapSpec(1, 0.08, 0), [1.08, 1.59, 2.13, 2.82]),
    4: ("GLL", "MG-CG", OverlapSpec(1, 0.08, 0), [1.34, 1.85, 2.24, 2.81]),
    5: ("GLL", "MG", OverlapSpec(1, 0.5, 0), [2.26, 2.76, 3.18, 3.66]),
    6: ("GLL", "MG-CG", OverlapSpec(1, 0.5, 0), [2.29, 2.67, 3.08, 3.75]),
    7: ("GL", "MG", OverlapSpec(0, 1, 0), [0.73, 0.96, 0.73, 0.40]),
    8: ("GL", "MG-CG", OverlapSpec(0, 1, 0), [1.49, 1.26, 1.07, 0.78]),
    9: ("GL", "MG", OverlapSpec(1, 0.08, 0), [0.73, 1.15, 1.70, 2.20]),
    10: ("GL", "MG-CG", OverlapSpec(1, 0.08, 0), [1.14, 1.38, 1.84, 2.15]),
    11: ("GL", "MG", OverlapSpec(1, 0.5, 0), [1.83, 2.28, 1.52, 0.94]),
    12: ("GL", "MG-CG", OverlapSpec(1, 0.5, 0), [1.90, 2.34, 1.88, 1.37]),
    13: ("GL", "MG", OverlapSpec(1, 0.09, 1), [1.36, 1.75, 1.87, 2.21]),
    14: ("GL", "MG-CG", OverlapSpec(1, 0.09, 1), [1.49, 1.81, 2.03, 2.22]),
}


def run_case(basis, solver, ov, P, ne, maxit=60):
    L = 2 * math.pi
    g = DG((ne, ne, ne), (L, L, L), P, 0 if basis == "GLL" else 1, 2.0, ov)
    N = g.ndofs()
    f = g.rhs_sin(3.0, 1.0, 1.0, 1.0)
    u = torch.from_numpy(uniform_vector(N, 3)).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if solver == "MG-CG":
        _, hist, ok = g.pcg_solve(u, f, rtol=1e-10, maxit=maxit)
        hist = list(hist)
    else:
        r = g.residual(u, f)
        hist = [math.sqrt(g.dot(r, r))]
        for _ in range(maxit):
            g.pmg_vcycle(u, f)
            r = g.residual(u, f)
            hist.append(math.sqrt(g.dot(r, r)))
            if hist[-1] <= 1e-10 * hist[0] or not math.isfinite(hist[-1]) or hist[-1] > 1e3 * hist[0]:
                break
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    n = len(hist) - 1
    rho = (hist[-1] / hist[0]) ** (1.0 / n) if n > 0 and hist[-1] > 0 else float("nan")
    # t_C: device time of one V(1,1) cycle (graph replay), tau10 = -10 t_C / lg rho per unknown
    # (the paper: ~3.5 us per unknown on one 3.1 GHz Broadwell core)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.pmg_vcycle(u, f)
    e0.record()
    for _ in range(5):
        g.pmg_vcycle(u, f)
    e1.record()
    torch.cuda.synchronize()
    t_c = e0.elapsed_time(e1) / 5 / 1e3
    tau10 = -10.0 * t_c / math.log10(rho) / N if 0 < rho < 1 else float("nan")
    no = [g.level_overlap(l)[0][0] for l in range(1, g.L + 1)]
    del g
    torch.cuda.empty_cache()
    return {"rho": rho, "lg": -math.log10(rho) if rho > 0 else None, "cycles": n, "hist": hist,
            "n_o": no, "dofs": N, "seconds": dt, "t_cycle_s": t_c, "tau10_ns_per_dof": tau10 * 1e9}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    rows = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else sorted(PAPER)
    Ps = [4, 8, 16, 32]
    out = {}
    for row in rows:
        basis, solver, ov, paper = PAPER[row]
        for P in Ps:
            ne = 128 // P
            res = run_case(basis, solver, ov, P, ne)
            out["%d/%d" % (row, P)] = dict(res, paper=paper[Ps.index(P)], basis=basis, solver=solver)
            print("row %2d P=%2d ne=%2d  -lg rho = %5.2f (paper %4.2f)  cycles %3d  n_o %s  t_C %.3f ms  tau10 %.2f ns/DOF" % (
                row, P, ne, res["lg"] or float("nan"), paper[Ps.index(P)], res["cycles"], res["n_o"],
                res["t_cycle_s"] * 1e3, res["tau10_ns_per_dof"]), flush=True)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "%s_table1_gpu.json" % tag), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
