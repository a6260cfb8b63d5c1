#!/usr/bin/env python
"""NEXT row f4: O(h^{P+1}) convergence of the GPU solve for the smooth periodic manufactured
solution u = sin x sin y sin z on [0, 2pi]^3 (north_star; BASELINE.json c2; SPEC.md:206, :521 —
the paper's own manufactured solution is garbled, DESIGN R14).

For each (basis, P) the mesh is refined N_e = k^3, the system A u = M f (f = 3 u) is solved on the
GPU by MG-CG (one V(1,1) per inexact-CG step) to ||r||/||r_0|| <= 1e-13, and the
nodal max error and the quadrature (mass-weighted) L2 error against the exact u are recorded with
the observed order lg2(e_k / e_2k).  Also reports n_10 and tau_10 of the solve.
Node coordinates come from the library's own 1D node table (dg_get_table which = 7); nothing here
touches oracle/.  Writes gpurun_out/<tag>_convergence_order.{json,txt}."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_1612_04796_b200 import DG
from workloads.configs import OverlapSpec

CASES = [  # (basis, P, [k...], overlap) — Table 1 row 3 (GLL) / row 13 (GL) overlaps
    ("GLL", 2, [4, 8, 16, 32], OverlapSpec(1, 0.08, 0)),
    ("GLL", 4, [4, 8, 16, 32], OverlapSpec(1, 0.08, 0)),
    ("GL", 4, [4, 8, 16, 32], OverlapSpec(1, 0.09, 1)),
    ("GLL", 8, [3, 6, 12, 24], OverlapSpec(1, 0.08, 0)),
    ("GL", 8, [3, 6, 12, 24], OverlapSpec(1, 0.09, 1)),
    ("GLL", 16, [3, 6, 12], OverlapSpec(1, 0.08, 0)),
]


def exact_and_mass(g, ne, P):
    """Exact nodal values of sin x sin y sin z and the diagonal mass in the library's
    element-major layout (e = ex + nx (ey + ny ez), node i + n (j + n k))."""
    n = P + 1
    L = 2 * math.pi
    xi = g.table(g.L, 0, 7)                       # reference nodes on [-1, 1]
    m1 = g.table(g.L, 0, 0)                       # 1D mass (quadrature weight * Delta / 2)
    h = L / ne
    x1 = (np.arange(ne)[:, None] + 0.5 * (xi[None, :] + 1.0)) * h      # (ne, n)
    s = np.sin(x1)
    # u[ez, ey, ex, k, j, i]
    u = (s[:, None, None, :, None, None] * s[None, :, None, None, :, None]
         * s[None, None, :, None, None, :])
    w = (m1[None, None, None, :, None, None] * m1[None, None, None, None, :, None]
         * m1[None, None, None, None, None, :]) * np.ones((ne, ne, ne, 1, 1, 1))
    return u.reshape(-1), w.reshape(-1)


def solve(basis, P, k, ov):
    L = 2 * math.pi
    g = DG((k, k, k), (L, L, L), P, 0 if basis == "GLL" else 1, 2.0, ov)
    N = g.ndofs()
    f = g.rhs_sin(3.0, 1.0, 1.0, 1.0)
    u = torch.zeros_like(f)
    g.pcg_solve(u, f, rtol=1e-13, maxit=60)       # warm-up: builds the solve's CUDA graph
    u.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    its, hist, ok = g.pcg_solve(u, f, rtol=1e-13, maxit=60)
    e1.record()
    torch.cuda.synchronize()
    hist = list(hist)
    ue, w = exact_and_mass(g, k, P)
    err = u.cpu().numpy() - ue
    err -= np.sum(w * err) / np.sum(w)            # the periodic solution is fixed up to a constant
    emax = float(np.max(np.abs(err)))
    el2 = float(math.sqrt(np.sum(w * err * err)))
    n = len(hist) - 1
    rho = (hist[-1] / hist[0]) ** (1.0 / n) if n else float("nan")
    t_it = e0.elapsed_time(e1) / 1e3 / max(n, 1)
    out = {"basis": basis, "P": P, "k": k, "dofs": N, "h": L / k, "err_max": emax, "err_l2": el2,
           "iters": n, "rho": rho, "n10": math.ceil(-10 / math.log10(rho)) if 0 < rho < 1 else None,
           "tau10_ns_per_dof": -10 * t_it / math.log10(rho) / N * 1e9 if 0 < rho < 1 else None,
           "converged": bool(ok)}
    del g
    torch.cuda.empty_cache()
    return out


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
    rows = []
    lines = ["| basis | P | N_e | DOF | max nodal error | order | L2 error | order | PCG its | n10 | tau10 ns/DOF |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for basis, P, ks, ov in CASES:
        prev = None
        for k in ks:
            r = solve(basis, P, k, ov)
            if prev is not None and r["err_max"] > 0:
                r["order_max"] = math.log2(prev["err_max"] / r["err_max"]) / math.log2(r["k"] / prev["k"])
                r["order_l2"] = math.log2(prev["err_l2"] / r["err_l2"]) / math.log2(r["k"] / prev["k"])
            rows.append(r)
            lines.append("| %s | %d | %d^3 | %d | %.3e | %s | %.3e | %s | %d | %s | %s |" % (
                basis, P, k, r["dofs"], r["err_max"],
                "%.2f" % r["order_max"] if "order_max" in r else "-", r["err_l2"],
                "%.2f" % r["order_l2"] if "order_l2" in r else "-", r["iters"], r["n10"],
                "%.2f" % r["tau10_ns_per_dof"] if r["tau10_ns_per_dof"] else "-"))
            print(lines[-1], flush=True)
            prev = r
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "%s_convergence_order.json" % tag), "w") as fh:
        json.dump(rows, fh, indent=1)
    with open(os.path.join(ROOT, "gpurun_out", "%s_convergence_order.txt" % tag), "w") as fh:
        fh.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
