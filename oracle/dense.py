"""O-dense — explicit IP-DG matrix from the 3D form, dense-LU Schwarz, pinned-LU coarse solve.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

O2  Global matrix A (PAPER.md:111-126 Eq. 4, :143-148 Eq. 6) assembled from the
    3D bilinear form with standard SIPG signs (reading R1, SURVEY C-1):
        a(u,v) = sum_e int_e grad u . grad v
               - sum_F int_F ( {d_n u}[v] + {d_n v}[u] ) + sum_F int_F mu [u][v]
    [v] = v^- - v^+ across a face with normal n^- pointing from "-" to "+",
    {w} = (w^- + w^+)/2, mu = penalty * P(P+1)/(2 Delta_normal): penalty times the
    stability threshold (reading R2).
    Volume: tensor GL/GLL quadrature at the (P+1)^3 collocation points;
    faces: tensor product of the two in-face 1D rules.  Periodic wrap.
O7  Subdomain solve: A_ss = A[I_s, I_s] (R_s A R_s^T literally, PAPER.md:204-213
    Eq. 9), dense LU (one factorisation reused for subdomains whose blocks are
    bitwise equal; equality asserted).
O8  Smoother step (Eq. 10): r = f - A u;
    du = sum_s R_s^T (W_s du_s); u += du.
O9  Coarse A_0^+ f_0 (Alg. 1 l.295): Euclidean projection of f_0,
    sparse LU with DOF 0 pinned, re-centre to Euclidean mean 0 (reading R9).
"""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import scipy.linalg as sla

from .basis import basis_data, stability_threshold
from .overlap import resolve_overlap, window_1d, weights_1d
from . import mg


def elem_index(ne, ex, ey, ez):
    nx, ny, nz = ne
    return (ex % nx) + nx * ((ey % ny) + ny * (ez % nz))


def assemble_A(ne, length, P, basis, penalty):
    """Explicit global IP-DG matrix (scipy CSR), element-major numbering."""
    nx, ny, nz = ne
    Ne = nx * ny * nz
    n = P + 1
    n3 = n ** 3
    bd = basis_data(basis, P)
    w, D = bd["w"], bd["D"]
    delta = [length[d] / ne[d] for d in range(3)]
    jac = delta[0] * delta[1] * delta[2] / 8.0
    I = sp.identity(n, format="csr")
    Dm = sp.csr_matrix(D)
    # gradient (reference) at the quadrature points, local index i + n j + n^2 k
    G = [sp.kron(I, sp.kron(I, Dm)), sp.kron(I, sp.kron(Dm, I)), sp.kron(Dm, sp.kron(I, I))]
    W3 = sp.diags(np.kron(w, np.kron(w, w)))
    Ke = sp.csr_matrix((n3, n3))
    for d in range(3):
        Ke = Ke + (jac * (2.0 / delta[d]) ** 2) * (G[d].T @ W3 @ G[d])
    Ke = sp.coo_matrix(Ke)
    rows = [((np.arange(Ne) * n3)[:, None] + Ke.row[None, :]).ravel()]
    cols = [((np.arange(Ne) * n3)[:, None] + Ke.col[None, :]).ravel()]
    vals = [np.tile(Ke.data, Ne)]

    # faces
    loc = np.arange(n3).reshape(n, n, n)          # [k, j, i]
    wz = w[:, None, None]; wy = w[None, :, None]; wx = w[None, None, :]
    ex, ey, ez = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ex, ey, ez = ex.ravel(), ey.ravel(), ez.ravel()
    e_minus = elem_index(ne, ex, ey, ez)
    for d, axis in ((0, 2), (1, 1), (2, 0)):
        # lines along direction d: rows = face points, columns = node along d
        lines = np.moveaxis(loc, axis, -1).reshape(n * n, n)
        other = [dd for dd in range(3) if dd != d]
        # face weight: product of the two in-face weights times the in-face Jacobian
        wf3 = wz * wy * wx
        wline = np.moveaxis(wf3, axis, -1).reshape(n * n, n)[:, 0] / w[0]
        wface = wline * (delta[other[0]] / 2.0) * (delta[other[1]] / 2.0)
        off = [0, 0, 0]; off[d] = 1
        e_plus = elem_index(ne, ex + off[0], ey + off[1], ez + off[2])
        mu = penalty * stability_threshold(P, delta[d])
        s = 2.0 / delta[d]
        Jv = np.concatenate([bd["phi_p"], -bd["phi_m"]])              # [u] = u^- - u^+
        Gv = 0.5 * s * np.concatenate([bd["dphi_p"], bd["dphi_m"]])   # {d_n u}
        F = -np.outer(Jv, Gv) - np.outer(Gv, Jv) + mu * np.outer(Jv, Jv)   # F[v, u]
        # global DOFs of the 2n line nodes for every (face, point)
        gm = e_minus[:, None, None] * n3 + lines[None, :, :]
        gp = e_plus[:, None, None] * n3 + lines[None, :, :]
        g = np.concatenate([gm, gp], axis=2)                      # (Ne, n^2, 2n)
        wfull = np.broadcast_to(wface[None, :, None, None], (Ne, n * n, 1, 1))
        vals.append((wfull * F[None, None, :, :]).ravel())
        rows.append(np.broadcast_to(g[:, :, :, None], (Ne, n * n, 2 * n, 2 * n)).ravel())
        cols.append(np.broadcast_to(g[:, :, None, :], (Ne, n * n, 2 * n, 2 * n)).ravel())
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(Ne * n3, Ne * n3)).tocsr()
    A.eliminate_zeros()
    return A


def mass_diag(ne, length, P, basis):
    """Diagonal GL/GLL mass M = J w_i w_j w_k."""
    n = P + 1
    w = basis_data(basis, P)["w"]
    delta = [length[d] / ne[d] for d in range(3)]
    jac = delta[0] * delta[1] * delta[2] / 8.0
    me = jac * np.kron(w, np.kron(w, w))
    return np.tile(me, ne[0] * ne[1] * ne[2])


def node_coords(ne, length, P, basis):
    """Physical coordinates (x, y, z) of every DOF, element-major."""
    n = P + 1
    x = basis_data(basis, P)["x"]
    delta = [length[d] / ne[d] for d in range(3)]
    nx, ny, nz = ne
    ez, ey, ex, k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx),
                                      np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    X = (ex + (x[i] + 1) / 2) * delta[0]
    Y = (ey + (x[j] + 1) / 2) * delta[1]
    Z = (ez + (x[k] + 1) / 2) * delta[2]
    return X.ravel(), Y.ravel(), Z.ravel()


def window_indices(ne, P, n_o):
    """Global DOF indices of every element-centred window, shape (Ne, m_x m_y m_z),
    window node (a, b, c) at a + m_x (b + m_y c)."""
    n = P + 1
    n3 = n ** 3
    nx, ny, nz = ne
    pos = [window_1d(0, P, n_o[d])[0] for d in range(3)]   # positions independent of basis
    offs = [np.array([p[0] for p in pos[d]]) for d in range(3)]
    locs = [np.array([p[1] for p in pos[d]]) for d in range(3)]
    ez, ey, ex = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ex, ey, ez = ex.ravel(), ey.ravel(), ez.ravel()      # subdomain s = element e (element-major)
    C, B, A_ = np.meshgrid(np.arange(len(locs[2])), np.arange(len(locs[1])), np.arange(len(locs[0])),
                           indexing="ij")
    A_, B, C = A_.ravel(), B.ravel(), C.ravel()
    e = elem_index(ne, ex[:, None] + offs[0][A_][None, :], ey[:, None] + offs[1][B][None, :],
                   ez[:, None] + offs[2][C][None, :])
    local = locs[0][A_] + n * (locs[1][B] + n * locs[2][C])
    return e * n3 + local[None, :]


class DenseLevel:
    def __init__(self, ne, length, P, basis, penalty, overlap):
        self.ne, self.length, self.P, self.basis = ne, length, P, basis
        self.n = P + 1
        self.A = assemble_A(ne, length, P, basis, penalty)
        self.N = self.A.shape[0]
        self.overlap = None
        if overlap is not None and P >= 2:
            deltas = [length[d] / ne[d] for d in range(3)]
            res = resolve_overlap(overlap.mode, overlap.value, overlap.floor, basis, P, deltas)
            self.overlap = res
            n_o = [r[0] for r in res]
            self.idx = window_indices(ne, P, n_o)
            W1 = [weights_1d(basis, P, r[0], r[1]) for r in res]
            self.W = np.kron(W1[2], np.kron(W1[1], W1[0]))
            self._factor()

    def _factor(self):
        """One LU per distinct (bitwise) block A_ss; congruent subdomains share it."""
        Ne, Mw = self.idx.shape
        self.lu_of = np.zeros(Ne, dtype=np.int64)
        blocks, lus = [], []
        for s in range(Ne):
            B = self.A[self.idx[s]][:, self.idx[s]].toarray()
            for t, Bt in enumerate(blocks):
                if np.array_equal(B, Bt):
                    self.lu_of[s] = t
                    break
            else:
                blocks.append(B)
                lus.append(sla.lu_factor(B))
                self.lu_of[s] = len(blocks) - 1
        self.lus = lus

    def apply(self, u):
        return self.A @ u

    def subdomain_solves(self, r):
        """du_s = A_ss^{-1} r_s for every subdomain: array (Ne, Mw)."""
        R = r[self.idx]
        out = np.empty_like(R)
        for t, lu in enumerate(self.lus):
            sel = np.nonzero(self.lu_of == t)[0]
            if len(sel):
                out[sel] = sla.lu_solve(lu, R[sel].T).T
        return out

    def smooth(self, u, f, steps):
        for _ in range(steps):
            r = f - self.A @ u
            du_s = self.subdomain_solves(r)
            du = np.bincount(self.idx.ravel(), weights=(du_s * self.W[None, :]).ravel(),
                             minlength=self.N)
            u = u + du
        return u


class DenseCoarse:
    """A_0^+ by pinned sparse LU (O9)."""

    def __init__(self, A0):
        self.N = A0.shape[0]
        self.lu = spla.splu(sp.csc_matrix(A0[1:, 1:]))

    def solve(self, f0):
        f = f0 - f0.mean()
        x = np.zeros(self.N)
        x[1:] = self.lu.solve(f[1:])
        return x - x.mean()


class DenseHierarchy(mg.Hierarchy):
    def __init__(self, ne, length, P, basis, penalty=2.0, overlap=None):
        super().__init__(ne, length, P, basis, penalty)
        self.levels = [DenseLevel(ne, length, Pl, basis, penalty, overlap if l > 0 else None)
                       for l, Pl in enumerate(self.Pl)]
        self.coarse_solver = DenseCoarse(self.levels[0].A)

    def apply(self, l, u):
        return self.levels[l].apply(u)

    def smooth(self, l, u, f, steps):
        return self.levels[l].smooth(u, f, steps)

    def coarse(self, f0):
        return self.coarse_solver.solve(f0)
