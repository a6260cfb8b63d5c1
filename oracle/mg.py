"""O4 transfers, O10 V-cycle (Algorithm 1), O11 inexact PCG, O12 metrics.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Levels P_l = 2^l, l = 0..L (§3.2); A_l re-discretised at P_l.
* Prolongation u_l += I_l u_{l-1} with the embedded interpolation
  I_l[i, j] = phi_j^{(P_{l-1})}(xi_i^{(P_l)}) applied along x, y, z per element;
  residual restriction with its transpose.
* V-cycle exactly as Algorithm 1; no mean anchoring (R10).
* Inexact PCG after Golub & Ye:
  alpha = <z,r>/<p,Ap>, beta = <z_new, r_new - r_old>/<z_old, r_old>,
  z = one V-cycle applied to r from a zero initial guess.
* rho = (r_n / r_0)^{1/n}, Euclidean residual norm; n10 = ceil(-10 / lg rho)
  (PAPER.md:337-349).
"""
import math
import numpy as np

from .basis import interp_matrix


class Hierarchy:
    """Level bookkeeping shared by the dense and matrix-free oracles."""

    def __init__(self, ne, length, P, basis, penalty):
        if P < 2 or (P & (P - 1)):
            raise ValueError("P must be a power of two >= 2 for multigrid (SPEC.md:323)")
        self.ne, self.length, self.P, self.basis, self.penalty = tuple(ne), tuple(length), P, basis, penalty
        self.L = int(round(math.log2(P)))
        self.Pl = [2 ** l for l in range(self.L + 1)]
        self.Ne = ne[0] * ne[1] * ne[2]
        self.I = [None] + [interp_matrix(basis, self.Pl[l - 1], self.Pl[l]) for l in range(1, self.L + 1)]

    def ndofs(self, l):
        return self.Ne * (self.Pl[l] + 1) ** 3

    def prolong(self, l, uc):
        I = self.I[l]
        nf, nc = I.shape
        U = uc.reshape(self.Ne, nc, nc, nc)                       # [e, c, b, a]
        return np.einsum("ia,jb,kc,ecba->ekji", I, I, I, U, optimize=True).ravel()

    def restrict(self, l, rf):
        I = self.I[l]
        nf, nc = I.shape
        R = rf.reshape(self.Ne, nf, nf, nf)                       # [e, k, j, i]
        return np.einsum("ia,jb,kc,ekji->ecba", I, I, I, R, optimize=True).ravel()

    # to be provided: apply(l, u), smooth(l, u, f, steps), coarse(f0)

    def schedule(self, nu1, nu2, growth=1):
        """Per-level smoothing counts (nu1, nu2) * growth^(L-l) (Table 2)."""
        s1 = [0] + [nu1 * growth ** (self.L - l) for l in range(1, self.L + 1)]
        s2 = [0] + [nu2 * growth ** (self.L - l) for l in range(1, self.L + 1)]
        return s1, s2


def vcycle(H, u, f, nu1=1, nu2=1, growth=1):
    """Algorithm 1."""
    s1, s2 = H.schedule(nu1, nu2, growth)
    L = H.L
    us = [None] * (L + 1)
    fs = [None] * (L + 1)
    us[L] = np.array(u, dtype=float, copy=True)          # l.284
    fs[L] = np.asarray(f, dtype=float)                    # l.285
    for l in range(L, 0, -1):                             # l.286
        if l < L:
            us[l] = np.zeros(H.ndofs(l))                  # l.287-289
        us[l] = H.smooth(l, us[l], fs[l], s1[l])          # l.290
        fs[l - 1] = H.restrict(l, fs[l] - H.apply(l, us[l]))   # l.292
    us[0] = H.coarse(fs[0])                               # l.295
    for l in range(1, L + 1):                             # l.298
        us[l] = us[l] + H.prolong(l, us[l - 1])           # l.299
        us[l] = H.smooth(l, us[l], fs[l], s2[l])          # l.301
    return us[L]                                          # l.304


def residual_norm(H, u, f):
    return float(np.linalg.norm(f - H.apply(H.L, u)))


def mg_solve(H, f, u0=None, rtol=1e-10, maxcycles=50, nu1=1, nu2=1, growth=1):
    """Repeated V-cycles until ||r_n||/||r_0|| <= rtol.  Returns (u, history)."""
    u = np.zeros_like(f) if u0 is None else np.array(u0, dtype=float)
    hist = [residual_norm(H, u, f)]
    for _ in range(maxcycles):
        if hist[-1] <= rtol * hist[0]:
            break
        u = vcycle(H, u, f, nu1, nu2, growth)
        hist.append(residual_norm(H, u, f))
    return u, hist


def pcg(H, f, u0=None, rtol=1e-10, maxit=100, nu1=1, nu2=1, growth=1, precond=None):
    """Inexact PCG (Golub-Ye) with one V-cycle as preconditioner.  Returns (u, history)."""
    if precond is None:
        precond = lambda r: vcycle(H, np.zeros_like(r), r, nu1, nu2, growth)
    u = np.zeros_like(f) if u0 is None else np.array(u0, dtype=float)
    r = f - H.apply(H.L, u)
    hist = [float(np.linalg.norm(r))]
    if hist[0] == 0.0:
        return u, hist
    z = precond(r)
    p = z.copy()
    zr = float(z @ r)
    for _ in range(maxit):
        q = H.apply(H.L, p)
        alpha = zr / float(p @ q)
        u = u + alpha * p
        r_new = r - alpha * q
        hist.append(float(np.linalg.norm(r_new)))
        if hist[-1] <= rtol * hist[0]:
            break
        z_new = precond(r_new)
        beta = float(z_new @ (r_new - r)) / zr
        p = z_new + beta * p
        r, z = r_new, z_new
        zr = float(z @ r)
    return u, hist


def rho(hist):
    n = len(hist) - 1
    return (hist[-1] / hist[0]) ** (1.0 / n)


def n10(rho_value):
    return int(math.ceil(-10.0 / math.log10(rho_value)))
