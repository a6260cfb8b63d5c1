"""NEXT row f3 on CPU: the element-slab schedule of paper_1612_04796_b200.slab
with world_size 2 over gloo.  The orchestration (which step, which halo exchange, in which order,
the gathered coarse solve, the all-reduced norm) is the product code; the numerical steps are
served here by a CPU stand-in built from the oracle's tables on each rank's LOCAL mesh (owned
layers + two ghost layers), so the two ranks together must reproduce the oracle's single-domain
V-cycles.  A missing or misplaced exchange leaves stale ghost layers and fails the comparison."""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleLocal:
    """CPU stand-in for binding.DG on a rank's local mesh: the same calls, served by oracle.mf
    (apply, transfers) and by the split of MFLevel.smooth into its two halves (window solves ->
    window buffer, weighted scatter-add)."""

    def __init__(self, ne, length, P, basis, penalty, overlap):
        from oracle.mf import MFHierarchy
        self.H = MFHierarchy(ne, length, P, basis, penalty, overlap)
        self.ne = tuple(ne)
        self.L = self.H.L
        self.Z = {}

    def level_overlap(self, l):
        lev = self.H.levels[l]
        no = [lev.overlap[d][0] for d in range(3)]
        return no, [lev.n + 2 * k for k in no]

    def residual(self, u, f, level, out):
        out.copy_(torch.from_numpy(f.numpy() - self.H.apply(level, u.numpy())))
        return out

    def schwarz_solve(self, r, level):
        from oracle.mf import to_lex
        lev = self.H.levels[level]
        R = to_lex(r.numpy(), lev.ne, lev.n)
        gx, gy, gz = lev.gidx
        Sx, Sy, Sz = lev.S
        lx, ly, lz = lev.lam
        inv = 1.0 / (lz[:, None, None] + ly[None, :, None] + lx[None, None, :])
        Wt = lev.W[2][:, None, None] * lev.W[1][None, :, None] * lev.W[0][None, None, :]
        T = R[gz[:, None, None, :, None, None], gy[None, :, None, None, :, None], gx[None, None, :, None, None, :]]
        T = T @ Sx
        T = np.swapaxes(np.swapaxes(T, -1, -2) @ Sy, -1, -2)
        T = np.moveaxis(np.moveaxis(T, -3, -1) @ Sz, -1, -3)
        T *= inv
        T = np.moveaxis(np.moveaxis(T, -3, -1) @ Sz.T, -1, -3)
        T = np.swapaxes(np.swapaxes(T, -1, -2) @ Sy.T, -1, -2)
        T = T @ Sx.T
        T *= Wt
        self.Z[level] = torch.from_numpy(np.ascontiguousarray(T).ravel())   # element-major windows

    def window_buffer(self, level):
        z = self.Z[level]
        return z, z.numel() // (self.ne[0] * self.ne[1] * self.ne[2])

    def schwarz_fold(self, u, zero, level):
        from oracle.mf import to_lex, from_lex
        lev = self.H.levels[level]
        gx, gy, gz = lev.gidx
        nz, ny, nx = (lev.ne[2] * lev.n, lev.ne[1] * lev.n, lev.ne[0] * lev.n)
        flat = ((gz[:, None, None, :, None, None] * ny + gy[None, :, None, None, :, None]) * nx
                + gx[None, None, :, None, None, :])
        T = self.Z[level].numpy().reshape(flat.shape)
        dG = np.bincount(flat.ravel(), weights=T.ravel(), minlength=nz * ny * nx).reshape(nz, ny, nx)
        du = torch.from_numpy(from_lex(dG, lev.ne, lev.n))
        if zero:
            u.copy_(du)
        else:
            u.add_(du)
        return u

    def restrict(self, rf, level, out):
        out.copy_(torch.from_numpy(self.H.restrict(level, rf.numpy())))
        return out

    def prolongate_add(self, uc, uf, level):
        uf.add_(torch.from_numpy(self.H.prolong(level, uc.numpy())))
        return uf

    def apply(self, u, level, out):
        out.copy_(torch.from_numpy(self.H.apply(level, u.numpy())))
        return out

    def axpby(self, y, a, x, b=1.0):
        y.copy_(a * x if b == 0.0 else a * x + b * y)
        return y

    def dot_range(self, x, y, count):
        return float(np.dot(x.numpy()[:count], y.numpy()[:count]))


class OracleCoarse:
    def __init__(self, ne, length, basis, penalty):
        from oracle.mf import MFHierarchy
        self.H = MFHierarchy(ne, length, 2, basis, penalty, None)

    def coarse_solve(self, f0):
        return torch.from_numpy(self.H.coarse(f0.numpy()))


CASES = {
    # name: (ne, length, P, basis, (overlap mode, value, floor))
    "gll-p4": ((3, 3, 6), (1.0, 1.0, 1.5), 4, 0, (1, 0.3, 1)),        # nz > nzl + 2: real ghosts
    "gl-p4-aniso": ((3, 4, 6), (2.0, 1.0, 1.5), 4, 1, (2, 0.2, 1)),
}


def _worker(rank, world, port, case, out):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1612_04796_b200.slab import SlabDG
    from workloads.configs import OverlapSpec
    from workloads import uniform_zero_mean
    ne, length, P, basis, ov = CASES[case]
    ov = OverlapSpec(*ov)
    nzl = ne[2] // world
    local_ne = (ne[0], ne[1], nzl + 2)
    local_len = (length[0], length[1], length[2] * (nzl + 2) / ne[2])
    sd = SlabDG(ne, length, P, basis, 2.0, ov, local=OracleLocal(local_ne, local_len, P, basis, 2.0, ov),
                coarse=OracleCoarse(ne, length, basis, 2.0), device="cpu")
    N = ne[0] * ne[1] * ne[2] * (P + 1) ** 3
    f = torch.from_numpy(uniform_zero_mean(N, 0))
    fl = sd.scatter_global(f)
    ul = torch.zeros_like(fl)
    iterates, norms = [], []
    for _ in range(2):
        sd.vcycle(ul, fl)
        iterates.append(sd.gather_global(ul).numpy().copy())
        r = sd.residual(ul, fl)
        norms.append(sd.dot(r, r))
    nex = sd.exchanges
    up = torch.zeros_like(fl)
    _, hist, ok = sd.pcg_solve(up, fl, rtol=1e-9, maxit=40)
    out[rank] = (iterates, norms, nex, sd.z0, sd.nzl, hist, ok, sd.gather_global(up).numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", sorted(CASES))
def test_two_rank_slab_vcycles_equal_single_domain_oracle(case):
    sys.path.insert(0, ROOT)
    from oracle.mf import MFHierarchy
    from oracle import mg
    from workloads.configs import OverlapSpec
    from workloads import uniform_zero_mean
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    ne, length, P, basis, ov = CASES[case]
    H = MFHierarchy(ne, length, P, basis, 2.0, OverlapSpec(*ov))
    f = uniform_zero_mean(H.ndofs(H.L), 0)
    u = np.zeros_like(f)
    for k in range(2):
        u = mg.vcycle(H, u, f)
        rn = mg.residual_norm(H, u, f) ** 2
        for r in range(world):
            iterates, norms, nex, z0, nzl = out[r][:5]
            assert np.max(np.abs(iterates[k] - u)) <= 1e-12 * np.max(np.abs(u)), (case, r, k)
            assert abs(norms[k] - rn) <= 1e-9 * rn
    # inexact PCG on slabs (all-reduced scalars) against the oracle's PCG on the whole mesh
    x_ref, h_ref = mg.pcg(H, f, rtol=1e-9, maxit=40)
    for r in range(world):
        hist, ok, x = out[r][5], out[r][6], out[r][7]
        assert ok and len(hist) == len(h_ref)
        assert np.allclose(hist, h_ref, rtol=1e-6)
        assert np.max(np.abs(x - x_ref)) <= 1e-8 * np.max(np.abs(x_ref))
    assert out[0][3] == 0 and out[1][3] == out[0][4]          # slabs are consecutive z ranges
    assert out[0][2] == out[1][2] > 0                         # both ranks issued the same exchanges


def test_slab_rejects_windows_spanning_the_periodic_line():
    sys.path.insert(0, ROOT)
    from paper_1612_04796_b200.slab import SlabDG
    from workloads.configs import OverlapSpec
    ov = OverlapSpec(0, 99, 0)                                # full overlap on every level
    local = OracleLocal((3, 3, 5), (1.0, 1.0, 5.0 / 3.0), 2, 0, 2.0, ov)
    with pytest.raises(ValueError):
        SlabDG((3, 3, 3), (1.0, 1.0, 1.0), 2, 0, 2.0, ov, local=local, coarse=None, device="cpu")
