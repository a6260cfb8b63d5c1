"""Diagnostic: run a few c3 V-cycles through a library built with -DPMG_PHASE_TIMING
(PMG_LIB=paper_1612_04796_b200/build/dbg/libpmgdg.so) so the Schwarz kernel prints per-phase
clock64() deltas for a sample of CTAs.  Not part of the product path."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1612_04796_b200 import DG
from workloads import get_config, uniform_zero_mean

c = get_config(sys.argv[1] if len(sys.argv) > 1 else "c3")
g = DG(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
f = torch.from_numpy(uniform_zero_mean(g.ndofs(), 0)).cuda()
u = torch.zeros_like(f)
g.set_graphs(False) if hasattr(g, "set_graphs") else None
for _ in range(2):
    g.pmg_vcycle(u, f)
torch.cuda.synchronize()
