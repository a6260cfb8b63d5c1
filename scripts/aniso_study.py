#!/usr/bin/env python
"""NEXT row f1: anisotropic study (Table 2).  Domains
(2 pi AR, 2 pi ceil(AR/2), 2 pi), 8^3 elements, P = 16 GLL, AR = 1..48, three methods:
(0.08 rel; 1,1 fix), (0.08 rel; 1,1 var), (0.08 max; 1,1 var) where var = (1,1) x 3^(L-l),
each as plain MG and as MG-CG.  Reports n10 = ceil(-10 / lg rho) per AR (the paper reports the
cycle count growing from 4 to 13 at AR = 48 for (0.08 max; 1,1 var))."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_1612_04796_b200 import DG
from workloads.configs import OverlapSpec
from workloads import uniform_vector

METHODS = {"rel-fix": (OverlapSpec(1, 0.08, 0), 1), "rel-var": (OverlapSpec(1, 0.08, 0), 3),
           "max-var": (OverlapSpec(2, 0.08, 0), 3)}


def run(AR, method, solver, P=16, ne=8, maxit=100):
    ov, growth = METHODS[method]
    L = (2 * math.pi * AR, 2 * math.pi * math.ceil(AR / 2), 2 * math.pi)
    g = DG((ne, ne, ne), L, P, 0, 2.0, ov)
    Lv = g.L
    nu = [0] + [growth ** (Lv - l) for l in range(1, Lv + 1)]
    g.set_schedule(nu, nu)
    N = g.ndofs()
    f = g.rhs_sin(3.0, 1.0 / AR, 1.0 / math.ceil(AR / 2), 1.0)
    u = torch.from_numpy(uniform_vector(N, 3)).cuda()
    if solver == "MG-CG":
        _, hist, _ = g.pcg_solve(u, f, rtol=1e-10, maxit=maxit)
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
    n = len(hist) - 1
    rho = (hist[-1] / hist[0]) ** (1.0 / n)
    n10 = math.ceil(-10 / math.log10(rho)) if 0 < rho < 1 else None
    no = [g.level_overlap(l)[0] for l in range(1, Lv + 1)]
    del g
    torch.cuda.empty_cache()
    return {"rho": rho, "n10": n10, "cycles": n, "n_o": no}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    ars = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8, 12, 16, 24, 32, 48]
    out = {}
    for solver in ("MG", "MG-CG"):
        for method in METHODS:
            for AR in ars:
                res = run(AR, method, solver)
                out["%s/%s/%d" % (solver, method, AR)] = res
                print("%-5s %-8s AR=%2d rho=%.3e n10=%s cycles=%d n_o(top)=%s" % (
                    solver, method, AR, res["rho"], res["n10"], res["cycles"], res["n_o"][-1]), flush=True)
    with open(os.path.join(ROOT, "gpurun_out", "%s_aniso_gpu.json" % tag), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
