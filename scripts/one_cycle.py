"""Two eager V(1,1) cycles (or one PCG solve for c5) of a config: the launch sequence the ncu
traffic capture (scripts/gpu_traffic.sh) measures; the second cycle is the steady state."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1612_04796_b200 import DG
from workloads import get_config, uniform_zero_mean

c = get_config(sys.argv[1])
g = DG(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
g.set_graphs(False)
f = g.rhs_sin(3.0, 1.0, 1.0, 1.0) if c.rhs == "sin" else torch.from_numpy(uniform_zero_mean(g.ndofs(), 0)).cuda()
u = torch.zeros_like(f)
n0 = g.launch_count()
g.pmg_vcycle(u, f)
n1 = g.launch_count()
g.pmg_vcycle(u, f)
torch.cuda.synchronize()
print("launches per cycle", n1 - n0, "second cycle", g.launch_count() - n1)
