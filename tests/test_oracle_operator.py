"""Pins for oracle O2 (explicit IP-DG matrix) and O-mf's 1D/Kronecker operator.

What pins what:
* symmetric PSD with a 1-D constant null space
* O2 (3D form) == Eq. 7 Kronecker form of 1D factors    PAPER.md:150-156 (two independent assemblies)
* SIPG consistency: A x^2 = M(-lap x^2) away from the seam   (catches sign errors in the face terms)
* scaling: A(s * domain) = s * A(domain)
* O(h^{P+1}) nodal convergence for the manufactured solution (north_star)
"""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import pytest

from oracle.basis import GLL, GL
from oracle.dense import assemble_A, mass_diag, node_coords
from oracle.mf import assemble_1d, to_lex, from_lex


@pytest.mark.parametrize("basis", [GLL, GL])
def test_symmetric_psd_nullspace(basis):
    A = assemble_A((3, 3, 3), (1.0, 1.0, 1.0), 2, basis, 2.0).toarray()
    assert np.max(np.abs(A - A.T)) < 1e-13 * np.max(np.abs(A))
    ev = np.linalg.eigvalsh(0.5 * (A + A.T))
    scale = ev[-1]
    assert abs(ev[0]) < 1e-12 * scale                 # constant null vector
    assert ev[1] > 1e-6 * scale                       # ... and only one
    assert np.max(np.abs(A @ np.ones(len(A)))) < 1e-12 * scale


@pytest.mark.parametrize("basis", [GLL, GL])
@pytest.mark.parametrize("P", [2, 3])
def test_eq7_kronecker_form(basis, P):
    ne, length = (3, 4, 3), (1.0, 2.5, 0.7)
    A = assemble_A(ne, length, P, basis, 2.0)
    n = P + 1
    L1, M1 = [], []
    for d in range(3):
        L, Mv = assemble_1d(basis, P, ne[d], length[d] / ne[d], 2.0)
        L1.append(sp.csr_matrix(L)); M1.append(sp.diags(Mv))
    Ak = (sp.kron(M1[2], sp.kron(M1[1], L1[0])) + sp.kron(M1[2], sp.kron(L1[1], M1[0]))
          + sp.kron(L1[2], sp.kron(M1[1], M1[0])))
    rng = np.random.default_rng(3)
    for _ in range(3):
        u = rng.standard_normal(A.shape[0])
        a = A @ u
        b = from_lex((Ak @ to_lex(u, ne, n).ravel()).reshape(ne[2] * n, ne[1] * n, ne[0] * n), ne, n)
        assert np.max(np.abs(a - b)) < 1e-12 * np.max(np.abs(a))


@pytest.mark.parametrize("basis", [GLL, GL])
@pytest.mark.parametrize("P", [2, 3, 4])
def test_sipg_consistency(basis, P):
    ne, length = (4, 3, 3), (1.0, 1.3, 0.9)
    A = assemble_A(ne, length, P, basis, 2.0)
    X, Y, Z = node_coords(ne, length, P, basis)
    M = mass_diag(ne, length, P, basis)
    n = P + 1
    e = np.repeat(np.arange(np.prod(ne)), n ** 3)
    ex, ey, ez = e % ne[0], (e // ne[0]) % ne[1], e // (ne[0] * ne[1])
    interior = (ex > 0) & (ex < ne[0] - 1) & (ey > 0) & (ey < ne[1] - 1) & (ez > 0) & (ez < ne[2] - 1)
    cases = [(X ** 2, -2.0 + 0 * X), (Z ** 2 * Y, -2.0 * Y)]
    if P >= 3:
        cases.append((Y ** 3, -6.0 * Y))
    for u, lap in cases:
        r = A @ u - M * lap
        assert np.max(np.abs(r[interior])) < 1e-11 * np.max(np.abs(M * lap) + 1)
        assert np.max(np.abs(r)) > 1e-3          # the seam rows do see the non-periodic jump


def test_scaling_invariance():
    a = assemble_A((3, 3, 3), (1.0, 1.0, 1.0), 3, GL, 2.0)
    b = assemble_A((3, 3, 3), (2.5, 2.5, 2.5), 3, GL, 2.0)
    assert abs(b - 2.5 * a).max() < 1e-12 * abs(a).max()


def _solve_manufactured(ne, P, basis):
    length = (1.0, 1.0, 1.0)
    A = assemble_A(ne, length, P, basis, 2.0).tocsc()
    X, Y, Z = node_coords(ne, length, P, basis)
    M = mass_diag(ne, length, P, basis)
    tp = 2 * np.pi
    ue = np.sin(tp * X) * np.sin(tp * Y) * np.sin(tp * Z)
    b = M * 3 * tp ** 2 * ue
    b -= b.mean()
    x, info = spla.cg(A.tocsr(), b, rtol=1e-13, maxiter=20000)
    assert info == 0
    assert np.linalg.norm(A @ x - b) < 1e-11 * np.linalg.norm(b)
    err = x - ue
    err -= np.sum(M * err) / np.sum(M)
    return np.sqrt(np.sum(M * err ** 2))


@pytest.mark.parametrize("basis", [GLL, GL])
@pytest.mark.parametrize("P", [2, 3])
def test_convergence_order(basis, P):
    # observed order between 6^3 and 12^3; theory h^{P+1} (GLL odd P superconverges nodally)
    order = np.log2(_solve_manufactured((6, 6, 6), P, basis) / _solve_manufactured((12, 12, 12), P, basis))
    assert P + 0.75 <= order <= P + 2.25, order


@pytest.mark.parametrize("basis", [GLL, GL])
@pytest.mark.parametrize("P", [1, 2, 4, 8, 16])
def test_stability_threshold(basis, P):
    """Reading R2: the coercivity threshold of the 1D SIPG matrix is P(P+1)/(2 Delta) exactly
    (PSD just above, indefinite just below) -- PAPER.md:331-333 defines mu_min as that threshold."""
    from oracle.basis import stability_threshold
    delta = 0.37
    thr = stability_threshold(P, delta)
    for fac, psd in ((1.0 + 1e-6, True), (1.0 - 1e-3, False)):
        mu_factor = fac            # penalty factor multiplies the threshold
        L, _ = assemble_1d(basis, P, 6, delta, mu_factor)   # even n_e: the alternating mode exists
        ev = np.linalg.eigvalsh(0.5 * (L + L.T))
        tol = 1e-10 * np.max(np.abs(ev))
        assert (ev[0] >= -tol) == psd, (fac, ev[:2])
    # penalty factor 2 (the paper's mu = 2 mu_min): one-dimensional null space, rest positive
    L, _ = assemble_1d(basis, P, 5, delta, 2.0)
    ev = np.linalg.eigvalsh(0.5 * (L + L.T))
    assert abs(ev[0]) < 1e-10 * ev[-1] and ev[1] > 1e-8 * ev[-1]
    assert thr == P * (P + 1) / (2 * delta)
