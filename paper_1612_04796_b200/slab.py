"""Element z-slab decomposition of the p-multigrid path over the ranks of a torch.distributed
group ("further acceleration, e.g. by parallelization").

One process per GPU.  Rank r owns the element layers ez in [r nz/R, (r+1) nz/R) of the periodic
nx x ny x nz mesh and works on a LOCAL mesh of nzl + 2 layers: its own layers plus one ghost layer
below and above (elements are stored e = ex + nx (ey + ny ez), so a layer of any element-major
vector is one contiguous range and a halo exchange is two plain sends and two receives).  Every
kernel is the single-GPU kernel of libpmgdg.so run on the local mesh (the periodic wrap between
the two ghost layers is never consumed); what the decomposition adds is WHEN ghost layers must
be refreshed.  One weighted Schwarz step (Eq. 10) on level l is

    exchange u ghosts           the residual of an owned element needs its neighbours' face traces
    r = f - A u                 (dg_residual; valid on owned layers)
    exchange r ghosts           the windows of owned subdomains reach n_o node layers into them
    Z = W A_ss^-1 R r           (dg_schwarz_solve; valid for owned subdomains)
    exchange Z ghosts           the fold of an owned element pulls from the neighbours' windows
    u += sum_s R_s^T Z_s        (dg_schwarz_fold; valid on owned layers)

The transfers are element-local; the restricted right-hand side gets its ghosts exchanged; the
coarse problem (8 DOF per element) is all-gathered and solved redundantly on every rank with the
global coarse pseudo-inverse (Alg. 1 l.295); residual norms and the scalars of the inexact PCG
 are all-reduced, its vector updates run through dg_axpby.  Arithmetic per owned
DOF is that of the single-GPU path (same kernels, same tables, same fold order).

This module is orchestration only (which ABI call and which exchange, in which order); the
local solver object `g` (binding.DG) and the global coarse solver `gc` run every numerical step.
Tests inject CPU stand-ins for g / gc to exercise the schedule with world_size 2 over gloo.
"""
import math


class SlabDG:
    def __init__(self, ne, length, P, basis, penalty=2.0, overlap=None, group=None, local=None,
                 coarse=None, device="cuda"):
        """ne, length: the GLOBAL mesh.  local / coarse: solver objects (tests); by default the
        CUDA library on the local extended mesh and on the global mesh (coarse solve only)."""
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        nx, ny, nz = ne
        if nz % self.world:
            raise ValueError("nz = %d must be a multiple of the world size %d" % (nz, self.world))
        self.ne, self.length, self.P = tuple(ne), tuple(length), P
        self.nzl = nz // self.world
        self.z0 = self.rank * self.nzl
        self.local_ne = (nx, ny, self.nzl + 2)
        self.local_length = (length[0], length[1], length[2] * (self.nzl + 2) / nz)
        self.device = device
        if local is None:
            from .binding import DG
            from workloads.configs import OverlapSpec
            local = DG(self.local_ne, self.local_length, P, basis, penalty, overlap)
            # the global P = 1 coarse operator: any hierarchy on the global mesh has it as level 0
            coarse = DG(self.ne, self.length, 2, basis, penalty, OverlapSpec(0, 1, 0))
        self.g, self.gc = local, coarse
        self.L = local.L
        self.n = [(1 << l) + 1 for l in range(self.L + 1)]
        for l in range(1, self.L + 1):
            # a window that covers the whole periodic z line (nz = 3 with full overlap) contains
            # the wrap coupling of the global operator, which no slab-local window can reproduce
            if local.level_overlap(l)[1][2] >= nz * self.n[l]:
                raise ValueError("level %d: the z window spans the whole periodic line (nz = %d); "
                                 "the slab decomposition needs nz >= 4 here" % (l, nz))
        self.nu1 = [1] * (self.L + 1)
        self.nu2 = [1] * (self.L + 1)
        self.layer = nx * ny                              # elements per z-layer
        self.exchanges = 0                                # halo exchanges issued (tests, bench)
        self._u = [self._empty(l) for l in range(self.L)]
        self._f = [self._empty(l) for l in range(self.L)]
        self._r = [self._empty(l) for l in range(self.L + 1)]

    # ---- layout ------------------------------------------------------------------------------
    def ndofs_local(self, level=None):
        level = self.L if level is None else level
        return self.layer * (self.nzl + 2) * self.n[level] ** 3

    def ndofs_owned(self, level=None):
        level = self.L if level is None else level
        return self.layer * self.nzl * self.n[level] ** 3

    def _empty(self, level):
        return self.torch.zeros(self.ndofs_local(level), dtype=self.torch.float64, device=self.device)

    def owned(self, v, per_elem):
        """View of the owned layers of a local vector with per_elem entries per element."""
        L = self.layer * per_elem
        return v[L: (self.nzl + 1) * L]

    def scatter_global(self, vglobal, level=None):
        """Local vector (ghosts filled) from a global element-major vector (any rank's copy)."""
        level = self.L if level is None else level
        per = self.n[level] ** 3
        L = self.layer * per
        nz = self.ne[2]
        layers = [(self.z0 - 1 + k) % nz for k in range(self.nzl + 2)]
        return self.torch.cat([vglobal[z * L: (z + 1) * L] for z in layers]).contiguous()

    def gather_global(self, vlocal, level=None):
        """Global vector from every rank's owned layers (all-gather)."""
        level = self.L if level is None else level
        own = self.owned(vlocal, self.n[level] ** 3).contiguous()
        if self.world == 1:
            return own.clone()
        out = self.torch.empty(own.numel() * self.world, dtype=own.dtype, device=own.device)
        self.dist.all_gather_into_tensor(out, own, group=self.group)
        return out

    # ---- halo exchange -----------------------------------------------------------------------
    def exchange(self, v, per_elem):
        """Refresh the two ghost layers of v (per_elem entries per element) from the z-neighbours:
        my lowest owned layer -> the lower neighbour's top ghost, my highest owned layer -> the upper
        neighbour's bottom ghost (periodic)."""
        L = self.layer * per_elem
        nzl = self.nzl
        lo_ghost, lo_own = v[0:L], v[L:2 * L]
        hi_own, hi_ghost = v[nzl * L:(nzl + 1) * L], v[(nzl + 1) * L:(nzl + 2) * L]
        self.exchanges += 1
        if self.world == 1:
            lo_ghost.copy_(hi_own)
            hi_ghost.copy_(lo_own)
            return
        dist = self.dist
        up, down = (self.rank + 1) % self.world, (self.rank - 1) % self.world
        ops = [dist.P2POp(dist.isend, lo_own, down, self.group, tag=0),
               dist.P2POp(dist.irecv, hi_ghost, up, self.group, tag=0),
               dist.P2POp(dist.isend, hi_own, up, self.group, tag=1),
               dist.P2POp(dist.irecv, lo_ghost, down, self.group, tag=1)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()

    # ---- Algorithm 1 on slabs ----------------------------------------------------------------
    def set_schedule(self, nu1, nu2):
        if len(nu1) != self.L + 1 or len(nu2) != self.L + 1:
            raise ValueError("set_schedule: nu1, nu2 need L+1 entries")
        self.nu1, self.nu2 = list(nu1), list(nu2)

    def residual(self, u, f, level=None, out=None):
        level = self.L if level is None else level
        self.exchange(u, self.n[level] ** 3)
        return self.g.residual(u, f, level=level, out=self._r[level] if out is None else out)

    def apply(self, u, out, level=None):
        level = self.L if level is None else level
        self.exchange(u, self.n[level] ** 3)
        return self.g.apply(u, level=level, out=out)

    def smooth(self, level, u, f, steps, zero):
        """`steps` weighted Schwarz iterations; zero: u == 0 on entry (r = f, Alg. 1 l.287-290;
        the ghosts of f must be valid)."""
        per = self.n[level] ** 3
        for it in range(steps):
            z = zero and it == 0
            if z:
                rin = f
            else:
                rin = self.residual(u, f, level)
                self.exchange(rin, per)
            self.g.schwarz_solve(rin, level=level)
            Z, mw = self.g.window_buffer(level)
            self.exchange(Z, mw)
            self.g.schwarz_fold(u, zero=z, level=level)
        if steps == 0 and zero:
            u.zero_()

    def coarse_solve(self, f0, out):
        """u_0 = A_0^+ f_0 on the GLOBAL P = 1 grid: all-gather, redundant solve, local extract."""
        fg = self.gather_global(f0, 0)
        ug = self.gc.coarse_solve(fg)
        out.copy_(self.scatter_global(ug, 0))
        return out

    def vcycle(self, u, f):
        """One V-cycle (Algorithm 1) in place on the local vector u; u and f are
        local vectors (owned layers + two ghost layers); on return the owned layers of u hold the
        new iterate."""
        L = self.L
        U, F = self._u + [u], self._f + [f]
        self.exchange(f, self.n[L] ** 3)
        for l in range(L, 0, -1):
            zero = l < L
            self.smooth(l, U[l], F[l], self.nu1[l], zero)
            r = self.residual(U[l], F[l], l)
            self.g.restrict(r, l, out=F[l - 1])
            self.exchange(F[l - 1], self.n[l - 1] ** 3)
        self.coarse_solve(F[0], U[0])
        for l in range(1, L + 1):
            self.g.prolongate_add(U[l - 1], U[l], l)
            self.smooth(l, U[l], F[l], self.nu2[l], False)
        return u

    # ---- norms and the V-cycle iteration ------------------------------------------------------
    def dot(self, x, y):
        """<x, y> over the owned layers, all-reduced over the ranks."""
        per = self.n[self.L] ** 3
        v = self.g.dot_range(self.owned(x, per), self.owned(y, per), self.ndofs_owned())
        if self.world > 1:
            t = self.torch.tensor([v], dtype=self.torch.float64, device=x.device)
            self.dist.all_reduce(t, group=self.group)
            v = float(t[0])
        return v

    def solve(self, u, f, rtol=1e-10, maxcycles=50):
        """V-cycles until ||r|| <= rtol ||r_0|| (Euclidean residual norm);
        returns (u, residual history, converged)."""
        r = self.residual(u, f)
        hist = [math.sqrt(self.dot(r, r))]
        for _ in range(maxcycles):
            if hist[-1] <= rtol * hist[0]:
                return u, hist, True
            self.vcycle(u, f)
            r = self.residual(u, f)
            hist.append(math.sqrt(self.dot(r, r)))
            if not math.isfinite(hist[-1]) or hist[-1] > 1e3 * hist[0]:
                return u, hist, False
        return u, hist, hist[-1] <= rtol * hist[0]

    # ---- inexact PCG (Golub-Ye), PAPER.md:309-311 ---------------------------------------------
    def pcg_solve(self, u, f, rtol=1e-10, maxit=100):
        """MG-preconditioned inexact CG on slabs: the library's recurrence (z = one V-cycle from
        zero, beta = <z, r - r_old> / <z_old, r_old>), dots all-reduced, vector updates through
        dg_axpby on the local vectors (ghost entries are refreshed by the next exchange).
        Returns (u, residual history, converged)."""
        g, torch = self.g, self.torch
        r = torch.empty_like(u)
        self.residual(u, f, out=r)
        hist = [math.sqrt(self.dot(r, r))]
        if hist[0] == 0.0:
            return u, hist, True
        z, p, q, rold = (torch.zeros_like(u) for _ in range(4))
        self.vcycle(z, r)
        g.axpby(p, 1.0, z, 0.0)
        zr_old = self.dot(z, r)
        for _ in range(maxit):
            self.apply(p, q)
            alpha = zr_old / self.dot(p, q)
            g.axpby(u, alpha, p, 1.0)
            g.axpby(rold, 1.0, r, 0.0)
            g.axpby(r, -alpha, q, 1.0)
            hist.append(math.sqrt(self.dot(r, r)))
            if not math.isfinite(hist[-1]) or hist[-1] > 1e3 * hist[0]:
                return u, hist, False
            if hist[-1] <= rtol * hist[0]:
                return u, hist, True
            g.axpby(z, 0.0, z, 0.0)                       # z = 0: V-cycle from a zero guess
            self.vcycle(z, r)
            zr = self.dot(z, r)
            beta = (zr - self.dot(z, rold)) / zr_old
            zr_old = zr
            g.axpby(p, 1.0, z, beta)
        return u, hist, False
