"""O-mf — matrix-free oracle: Eq. 7 Kronecker apply + fast-diagonalisation Schwarz.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Validated against O-dense
(oracle.dense) on small grids by tests/test_oracle_*.py; used for full-size
parity and as the timed CPU baseline (BASELINE.md "CPU baseline plan").

* 1D IP matrix: the periodic 1D SIPG form assembled with an explicit face loop
  (volume (2/Delta) sum_q w_q phi_i' phi_j' plus, per face, -{u'}[v] - {v'}[u]
  + mu [u][v]); M = (Delta/2) diag(w) (Eq. 7).
* Apply: A = Mz(x)My(x)Lx + Mz(x)Ly(x)Mx + Lz(x)My(x)Mx on the global
  lexicographic grid.
* Subdomain solve by fast diagonalisation:
  A_ss^{-1} = (Sz(x)Sy(x)Sx) (I(x)I(x)Lx + I(x)Ly(x)I + Lz(x)I(x)I)^{-1} (Sz^T(x)Sy^T(x)Sx^T),
  S^T M_s S = I, with the 1D restricted matrices taken as principal
  submatrices (Dirichlet truncation, R_s A R_s^T) of the periodic 1D L and M,
  and eigenpairs from mpmath.eigsy at 40 significant digits, then rounded
  (reading R4).
* Coarse A_0^+: Euclidean projection, global fast diagonalisation of the periodic
  P=1 Kronecker operator with the zero (constant) mode dropped, Euclidean
  re-centring (as O9; checked against O-dense's pinned LU and numpy pinv).
"""
from functools import lru_cache
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .basis import basis_data, stability_threshold
from .overlap import resolve_overlap, weights_1d
from . import mg


def assemble_1d(basis, P, ne, delta, penalty):
    """Periodic 1D SIPG matrix L (dense, ne*n square) and mass diagonal."""
    bd = basis_data(basis, P)
    n = P + 1
    N = ne * n
    L = np.zeros((N, N))
    s = 2.0 / delta
    Kv = s * bd["D"].T @ np.diag(bd["w"]) @ bd["D"]
    mu = penalty * stability_threshold(P, delta)
    for e in range(ne):
        L[e * n:(e + 1) * n, e * n:(e + 1) * n] += Kv
    Jv = np.concatenate([bd["phi_p"], -bd["phi_m"]])
    Gv = 0.5 * s * np.concatenate([bd["dphi_p"], bd["dphi_m"]])
    F = -np.outer(Jv, Gv) - np.outer(Gv, Jv) + mu * np.outer(Jv, Jv)
    for e in range(ne):                  # face between e (minus) and e+1 (plus), periodic
        idx = np.concatenate([e * n + np.arange(n), ((e + 1) % ne) * n + np.arange(n)])
        L[np.ix_(idx, idx)] += F
    Mv = np.tile(0.5 * delta * bd["w"], ne)
    return L, Mv


@lru_cache(maxsize=None)
def _eig_mp(key, Ls_bytes, Ms_bytes, m):
    import mpmath
    mpmath.mp.dps = 40
    Ls = np.frombuffer(Ls_bytes).reshape(m, m)
    Ms = np.frombuffer(Ms_bytes)
    isq = [1 / mpmath.sqrt(mpmath.mpf(float(x))) for x in Ms]
    B = mpmath.matrix(m, m)
    for i in range(m):
        for j in range(m):
            B[i, j] = isq[i] * mpmath.mpf(float(Ls[i, j])) * isq[j]
    # symmetrise exactly (Ls is symmetric up to assembly round-off)
    for i in range(m):
        for j in range(i + 1, m):
            a = (B[i, j] + B[j, i]) / 2
            B[i, j] = a
            B[j, i] = a
    E, Q = mpmath.eigsy(B)
    lam = np.array([float(E[i]) for i in range(m)])
    S = np.array([[float(isq[i] * Q[i, j]) for j in range(m)] for i in range(m)])
    order = np.argsort(lam)
    return lam[order], S[:, order]


def restricted_eig(Ls, Ms):
    """Generalized eigenpairs Ls S = diag(Ms) S Lambda, S^T diag(Ms) S = I (40-digit mpmath)."""
    Ls = np.ascontiguousarray(Ls, dtype=float)
    Ms = np.ascontiguousarray(Ms, dtype=float)
    return _eig_mp(None, Ls.tobytes(), Ms.tobytes(), len(Ms))


def to_lex(u, ne, n):
    nx, ny, nz = ne
    U = u.reshape(nz, ny, nx, n, n, n)                     # [ez, ey, ex, k, j, i]
    return U.transpose(0, 3, 1, 4, 2, 5).reshape(nz * n, ny * n, nx * n)


def from_lex(G, ne, n):
    nx, ny, nz = ne
    U = G.reshape(nz, n, ny, n, nx, n).transpose(0, 2, 4, 1, 3, 5)
    return np.ascontiguousarray(U).ravel()


class MFLevel:
    def __init__(self, ne, length, P, basis, penalty, overlap):
        self.ne, self.P, self.n = tuple(ne), P, P + 1
        self.delta = [length[d] / ne[d] for d in range(3)]
        self.L1, self.M1 = [], []
        for d in range(3):
            L, Mv = assemble_1d(basis, P, ne[d], self.delta[d], penalty)
            self.L1.append(sp.csr_matrix(L))
            self.M1.append(Mv)
            if d == 0:
                self._Ldense = [L]
            else:
                self._Ldense.append(L)
        self.N = int(np.prod(ne)) * self.n ** 3
        self.overlap = None
        if overlap is not None and P >= 2:
            res = resolve_overlap(overlap.mode, overlap.value, overlap.floor, basis, P, self.delta)
            self.overlap = res
            self.S, self.lam, self.W, self.gidx = [], [], [], []
            n = self.n
            for d in range(3):
                n_o = res[d][0]
                # window of the subdomain centred on element 1 (no wrap; ne >= 3)
                win = np.arange(n - n_o, 2 * n + n_o)
                Ls = self._Ldense[d][np.ix_(win, win)]
                lam, S = restricted_eig(Ls, self.M1[d][win])
                self.S.append(S)
                self.lam.append(lam)
                self.W.append(weights_1d(basis, P, n_o, res[d][1]))
                Nd = ne[d] * n
                self.gidx.append((np.arange(ne[d])[:, None] * n - n_o + np.arange(len(win))[None, :]) % Nd)

    def apply_lex(self, G):
        Mx, My, Mz = self.M1
        Lx, Ly, Lz = self.L1
        Z, Y, X = G.shape
        out = (Lx @ G.reshape(-1, X).T).T.reshape(Z, Y, X) * (Mz[:, None, None] * My[None, :, None])
        Gy = G.transpose(0, 2, 1).reshape(-1, Y)
        out += (Ly @ Gy.T).T.reshape(Z, X, Y).transpose(0, 2, 1) * (Mz[:, None, None] * Mx[None, None, :])
        out += (Lz @ G.reshape(Z, -1)).reshape(Z, Y, X) * (My[None, :, None] * Mx[None, None, :])
        return out

    def apply(self, u):
        return from_lex(self.apply_lex(to_lex(u, self.ne, self.n)), self.ne, self.n)

    def smooth(self, u, f, steps):
        ne, n = self.ne, self.n
        G = to_lex(u, ne, n)
        F = to_lex(f, ne, n)
        Z, Y, X = G.shape
        gx, gy, gz = self.gidx
        Sx, Sy, Sz = self.S
        lx, ly, lz = self.lam
        inv = 1.0 / (lz[:, None, None] + ly[None, :, None] + lx[None, None, :])
        Wt = self.W[2][:, None, None] * self.W[1][None, :, None] * self.W[0][None, None, :]
        iz = gz[:, None, None, :, None, None]
        iy = gy[None, :, None, None, :, None]
        ix = gx[None, None, :, None, None, :]
        flat = ((iz * Y + iy) * X + ix)
        for _ in range(steps):
            R = F - self.apply_lex(G)
            Rw = R[iz, iy, ix]                          # (nz, ny, nx, mz, my, mx) windows
            T = Rw @ Sx                                 # S_x^T along x
            T = np.swapaxes(np.swapaxes(T, -1, -2) @ Sy, -1, -2)
            T = np.moveaxis(np.moveaxis(T, -3, -1) @ Sz, -1, -3)
            T *= inv
            T = np.moveaxis(np.moveaxis(T, -3, -1) @ Sz.T, -1, -3)
            T = np.swapaxes(np.swapaxes(T, -1, -2) @ Sy.T, -1, -2)
            T = T @ Sx.T
            T *= Wt
            dG = np.bincount(np.broadcast_to(flat, T.shape).ravel(), weights=T.ravel(),
                             minlength=Z * Y * X).reshape(Z, Y, X)
            G = G + dG
        return from_lex(G, ne, n)


class MFCoarse:
    """A_0^+ f_0 by global fast diagonalisation of the periodic P=1 Kronecker operator
    (1D eigenpairs at 40 digits; the constant mode has eigenvalue 0 and is dropped) after
    the Euclidean projection of f_0, then Euclidean re-centring (O9, reading R9).  Pinned
    against the pinned-LU O-dense coarse solve and numpy.linalg.pinv by tests/."""

    def __init__(self, lev):
        self.lev = lev
        self.S, self.lam = [], []
        for d in range(3):
            lam, S = restricted_eig(lev.L1[d].toarray(), lev.M1[d])
            self.S.append(S)
            self.lam.append(lam)
        lx, ly, lz = self.lam
        den = lz[:, None, None] + ly[None, :, None] + lx[None, None, :]
        null = den <= 1e-12 * den.max()
        assert null.sum() == 1, "exactly one null mode expected"
        self.inv = np.where(null, 0.0, 1.0 / np.where(null, 1.0, den))

    def solve(self, f0):
        ne, n = self.lev.ne, self.lev.n
        G = to_lex(f0 - f0.mean(), ne, n)
        Sx, Sy, Sz = self.S
        T = np.einsum("cba,ai,bj,ck->kji", G, Sx, Sy, Sz, optimize=True) * self.inv
        X = np.einsum("kji,ai,bj,ck->cba", T, Sx, Sy, Sz, optimize=True)
        x = from_lex(X, ne, n)
        return x - x.mean()


class MFHierarchy(mg.Hierarchy):
    def __init__(self, ne, length, P, basis, penalty=2.0, overlap=None):
        super().__init__(ne, length, P, basis, penalty)
        self.levels = [MFLevel(ne, length, Pl, basis, penalty, overlap if l > 0 else None)
                       for l, Pl in enumerate(self.Pl)]
        self.coarse_solver = MFCoarse(self.levels[0])

    def apply(self, l, u):
        return self.levels[l].apply(u)

    def smooth(self, l, u, f, steps):
        return self.levels[l].smooth(u, f, steps)

    def coarse(self, f0):
        return self.coarse_solver.solve(f0)
