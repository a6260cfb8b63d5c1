"""Diagnostic: V-cycles, applies and a PCG solve on small meshes with the window shapes and
polynomial degrees of every config (so every compile-time kernel runs at small grids, including
the ragged 3x3x4 element grids), e.g. `python scripts/small_mesh_probe.py` on a GPU box.
(compute-sanitizer is not available on the GPU pool.)  Not part of the product path."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1612_04796_b200 import DG
from workloads import get_config, uniform_zero_mean

CASES = [("c1", None), ("c2", (4, 4, 4)), ("c3", (3, 3, 4)), ("c4", (3, 3, 3)), ("c5", (4, 3, 3))]
for name, ne in CASES[: int(os.environ.get("PMG_SAN_CASES", len(CASES)))]:
    c = get_config(name)
    ne = ne or c.ne
    length = c.length
    g = DG(ne, length, c.P, c.basis, c.penalty, c.overlap)
    N = g.ndofs()
    f = torch.from_numpy(uniform_zero_mean(N, 0)).cuda()
    u = torch.zeros_like(f)
    g.pmg_vcycle(u, f)
    g.pmg_vcycle(u, f)
    v = g.apply(u)
    u2 = torch.zeros_like(f)
    _, hist, _ = g.pcg_solve(u2, f, rtol=1e-6, maxit=30)
    torch.cuda.synchronize()
    print(name, ne, "N", N, "|u|", float(u.norm()), "|Au|", float(v.norm()), "pcg its", len(hist) - 1, flush=True)
