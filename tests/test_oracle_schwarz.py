"""Pins for oracle O5-O8 (overlap, weights, subdomain solves, smoother) and O-mf's FDM.

* overlap layer counts == Table 1 n_o column, golden file
* partition of unity sum_s R_s^T W_s R_s = I on every level
* hat shape: 0 at the subdomain boundary, 1 on the non-overlapped core, q(1/2)=1/2 (Fig. 2)
* FDM (O-mf) == dense LU (O-dense) subdomain solves; S^T M S = I, S^T L S = Lambda
* smoother fixed point
"""
import os
import numpy as np
import pytest

from oracle.basis import GLL, GL, nodes_weights
from oracle.overlap import (resolve_overlap, weights_1d, hat_weight, quintic, window_1d,
                            OVL_NODES, OVL_REL, OVL_MAXREL)
from oracle.dense import DenseLevel, window_indices
from oracle.mf import MFLevel
from workloads import CONFIGS, get_config
from workloads.configs import OverlapSpec

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_table1_overlap_sequences():
    rows = [l.split("#")[0].split() for l in open(os.path.join(GOLDEN, "table1_overlap_layers.txt"))]
    rows = [r for r in rows if r]
    assert len(rows) == 5
    for row, kind, alpha, floor, *seq in rows:
        b = GLL if kind == "GLL" else GL
        got = [resolve_overlap(OVL_REL, float(alpha), int(floor), b, P, [1.0, 1.0, 1.0])[0][0]
               for P in (2, 4, 8, 16, 32)]
        assert got == [int(s) for s in seq], (row, got, seq)


def test_maxrelative_c5_layers():
    # Table 2 "0.08 max" on c5's box: Delta = (3, 1/16, 1/16)
    deltas = [3.0, 1.0 / 16, 1.0 / 16]
    got = {P: [r[0] for r in resolve_overlap(OVL_MAXREL, 0.08, 1, GL, P, deltas)] for P in (2, 4, 8)}
    assert got == {2: [1, 3, 3], 4: [1, 5, 5], 8: [1, 9, 9]}


def test_hat_shape():
    assert quintic(0.5) == 0.5 and quintic(0.0) == 0.0 and quintic(1.0) == 1.0
    t = np.linspace(0, 1, 101)
    assert np.allclose(quintic(t) + quintic(1 - t), 1.0, atol=1e-15)
    h = 0.3
    assert hat_weight(1 + h, h) == 0.0                       # subdomain boundary
    assert np.all(hat_weight(np.linspace(-(1 - h), 1 - h, 11), h) == 1.0)   # non-overlapped core
    assert abs(hat_weight(1.0, h) - 0.5) < 1e-15 and abs(hat_weight(-1.0, h) - 0.5) < 1e-15
    # FixedNodes(1)/Relative(0.08) GLL at P=4: face DOFs 1/2, everything else 1 (SURVEY C-6)
    for mode, val in ((OVL_NODES, 1), (OVL_REL, 0.08)):
        n_o, dref = resolve_overlap(mode, val, 0, GLL, 4, [1, 1, 1])[0]
        w = weights_1d(GLL, 4, n_o, dref)
        assert np.allclose(w, [0.5, 0.5, 1, 1, 1, 0.5, 0.5])


def _levels_of(cfg, ne):
    c = get_config(cfg, ne)
    P = c.P
    out = []
    while P >= 2:
        out.append((c, P))
        P //= 2
    return out


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_partition_of_unity(cfg):
    for c, P in _levels_of(cfg, 3):
        deltas = [c.length[d] / c.ne[d] for d in range(3)]
        res = resolve_overlap(c.overlap.mode, c.overlap.value, c.overlap.floor, c.basis, P, deltas)
        idx = window_indices(c.ne, P, [r[0] for r in res])
        W1 = [weights_1d(c.basis, P, r[0], r[1]) for r in res]
        W = np.kron(W1[2], np.kron(W1[1], W1[0]))
        s = np.bincount(idx.ravel(), weights=np.broadcast_to(W, idx.shape).ravel(),
                        minlength=c.nelem * (P + 1) ** 3)
        assert np.max(np.abs(s - 1.0)) < 1e-14, (cfg, P)


@pytest.mark.parametrize("cfg,ne", [("c1", 4), ("c2", 3), ("c5", 3), ("c3", 3)])
def test_fdm_equals_dense_lu(cfg, ne):
    c = get_config(cfg, ne)
    rng = np.random.default_rng(7)
    for _, P in _levels_of(cfg, ne):
        if (P + 1) ** 3 * 8 > 2500 and cfg in ("c3",) and P > 4:
            continue                     # dense LU of 23^3 windows is too slow for the CPU suite
        if cfg == "c5" and P > 4:
            continue
        d = DenseLevel(c.ne, c.length, P, c.basis, c.penalty, c.overlap)
        m = MFLevel(c.ne, c.length, P, c.basis, c.penalty, c.overlap)
        u = rng.uniform(-1, 1, d.N)
        f = rng.uniform(-1, 1, d.N)
        a, b = d.smooth(u, f, 1), m.smooth(u, f, 1)
        # both are exact solvers; their forward-error difference is bounded by cond(A_ss)*eps
        Ass = d.A[d.idx[0]][:, d.idx[0]].toarray()
        tol = max(1e-13, 50 * np.finfo(float).eps * np.linalg.cond(Ass))
        assert np.max(np.abs(a - b)) <= tol * np.max(np.abs(a)), (cfg, P, tol)


@pytest.mark.parametrize("basis,P,n_o", [(GLL, 16, 3), (GLL, 32, 6), (GL, 8, 9), (GL, 8, 1)])
def test_fdm_eigenpairs(basis, P, n_o):
    from oracle.mf import assemble_1d, restricted_eig
    n = P + 1
    for delta in (1.0 / 16, 3.0):
        L, Mv = assemble_1d(basis, P, 4, delta, 2.0)
        win = np.arange(n - n_o, 2 * n + n_o)
        Ls, Ms = L[np.ix_(win, win)], Mv[win]
        lam, S = restricted_eig(Ls, Ms)
        m = len(win)
        assert np.max(np.abs(S.T @ (Ms[:, None] * S) - np.eye(m))) < 1e-13
        assert np.max(np.abs(S.T @ Ls @ S - np.diag(lam))) < 1e-13 * lam[-1]
        assert lam[0] > 0                                    # A_ss regular
        # FDM inverse of a 2-direction Kronecker sum vs dense solve (forward error)
        A2 = np.kron(np.diag(Ms), Ls) + np.kron(Ls, np.diag(Ms))
        r = np.random.default_rng(1).standard_normal(m * m)
        x_ref = np.linalg.solve(A2, r)
        T = S.T @ r.reshape(m, m) @ S
        T /= lam[:, None] + lam[None, :]
        x = (S @ T @ S.T).ravel()
        assert np.max(np.abs(x - x_ref)) < 1e-12 * np.max(np.abs(x_ref)) * max(1, P / 8)


def test_smoother_fixed_point():
    c = get_config("c1")
    d = DenseLevel(c.ne, c.length, 4, c.basis, c.penalty, c.overlap)
    u = np.random.default_rng(2).uniform(-1, 1, d.N)
    f = d.apply(u)
    assert np.max(np.abs(d.smooth(u, f, 2) - u)) < 1e-12


def test_quintic_is_the_c2_smoothstep():
    """Fig. 2 caption: "piece-wise quintic transition from 0 ... to 1".  A quintic
    has six coefficients; q(0) = 0, q(1) = 1 and vanishing first and second derivatives at both
    ends (C^2 contact with the constant pieces) determine it uniquely.  Solve those six conditions
    and compare with the oracle's transition on a grid (a dropped term or a wrong coefficient in
    oracle.overlap.quintic fails this)."""
    def row(t, der):
        # d^der/dt^der of (1, t, ..., t^5) at t
        r = np.zeros(6)
        for k in range(der, 6):
            c = 1.0
            for j in range(der):
                c *= (k - j)
            r[k] = c * t ** (k - der)
        return r
    A = np.array([row(0, 0), row(0, 1), row(0, 2), row(1, 0), row(1, 1), row(1, 2)])
    coef = np.linalg.solve(A, np.array([0, 0, 0, 1, 0, 0], dtype=float))
    t = np.linspace(-0.25, 1.25, 61)
    want = np.polynomial.polynomial.polyval(np.clip(t, 0, 1), coef)
    assert np.max(np.abs(quintic(t) - want)) < 1e-14
