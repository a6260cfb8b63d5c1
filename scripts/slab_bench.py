#!/usr/bin/env python
"""NEXT row f3: V(1,1) cycles through the element-slab path (paper_1612_04796_b200.slab.SlabDG).
Single process: one rank whose ghost layers are its own periodic images (measures the cost of the
ghost layers, the exchanges and the eager orchestration against the plain graph-replayed cycle).
Under torchrun (--nproc-per-node N, NCCL): N ranks, strong scaling of one global mesh.
usage: python scripts/slab_bench.py [config] [cycles]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import torch.distributed as dist

from paper_1612_04796_b200 import DG, SlabDG
from workloads import get_config, uniform_zero_mean


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    c = get_config(name)
    sd = SlabDG(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    f = torch.from_numpy(uniform_zero_mean(c.ndofs, 0)).cuda()
    fl = sd.scatter_global(f)
    ul = torch.zeros_like(fl)
    _, hist, _ = sd.solve(ul, fl, rtol=1e-10, maxcycles=3)          # warm-up + residual history
    ex0 = sd.exchanges
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record()
    for _ in range(cycles):
        sd.vcycle(ul, fl)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / cycles
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    out = {"config": name, "world": world, "ms_per_cycle": ms, "dof_per_s": c.ndofs / (ms * 1e-3),
           "exchanges_per_cycle": (sd.exchanges - ex0) / cycles, "local_mesh": sd.local_ne,
           "residual_history": hist}
    if world == 1:
        g = DG(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
        u = torch.zeros_like(f)
        for _ in range(3):
            g.pmg_vcycle(u, f)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(cycles):
            g.pmg_vcycle(u, f)
        e1.record()
        torch.cuda.synchronize()
        out["plain_ms_per_cycle"] = e0.elapsed_time(e1) / cycles
    if sd.rank == 0:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
