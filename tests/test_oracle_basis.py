"""Pins for oracle O1 (basis) and the penalty formula against the paper/SPEC and mathematics."""
import math
import os
import numpy as np
import pytest

from oracle.basis import (GLL, GL, nodes_weights, basis_data, interp_matrix, face_distances,
                          penalty_min, lagrange)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#")[0].strip()
        if line:
            rows.append(line.split())
    return rows


def test_spec_basis_examples():
    for kind, P, q, *vals in _golden("basis_examples.txt"):
        b = GLL if kind == "GLL" else GL
        P = int(P)
        vals = np.array([float(v) for v in vals])
        x, w = nodes_weights(b, P)
        got = {"nodes": x, "weights": w, "facedist": face_distances(b, P)}[q]
        assert np.allclose(got, vals, rtol=0, atol=1e-14), (kind, P, q, got)


@pytest.mark.parametrize("basis", [GLL, GL])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 7, 8, 16, 32])
def test_quadrature_exactness(basis, P):
    x, w = nodes_weights(basis, P)
    deg = 2 * P - 1 if basis == GLL else 2 * P + 1
    assert np.all(np.diff(x) > 0) and np.allclose(x, -x[::-1], atol=1e-15)
    for k in range(deg + 1):
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.sum(w * x ** k) - exact) < 2e-14, (k,)
    # one degree higher is NOT integrated exactly (the rule is not accidentally stronger)
    if P <= 8:
        k = deg + 1
        assert abs(np.sum(w * x ** k) - 2.0 / (k + 1)) > 1e-8


@pytest.mark.parametrize("basis", [GLL, GL])
@pytest.mark.parametrize("P", [1, 2, 5, 8, 16])
def test_derivative_exactness(basis, P):
    bd = basis_data(basis, P)
    x, D = bd["x"], bd["D"]
    for k in range(P + 1):
        got = D @ x ** k
        ref = k * x ** (k - 1) if k else np.zeros_like(x)
        assert np.max(np.abs(got - ref)) < 1e-11 * max(1.0, k * k)
    # traces: phi(+-1) reproduce polynomials at the end points, phi' their derivatives
    for k in range(P + 1):
        assert abs(bd["phi_p"] @ x ** k - 1.0) < 1e-12
        assert abs(bd["phi_m"] @ x ** k - (-1.0) ** k) < 1e-12
        assert abs(bd["dphi_p"] @ x ** k - k) < 1e-10 * max(1, k * k)


def test_gll_p8_smallest_face_distance():
    d = face_distances(GLL, 8)
    assert d[0] == 0.0 and abs(d[1] - 0.1002) < 5e-5


@pytest.mark.parametrize("basis", [GLL, GL])
def test_interpolation_reproduces_polynomials(basis):
    for Pc, Pf in ((1, 2), (2, 4), (4, 8), (8, 16), (16, 32)):
        I = interp_matrix(basis, Pc, Pf)
        xc, _ = nodes_weights(basis, Pc)
        xf, _ = nodes_weights(basis, Pf)
        assert np.allclose(I.sum(axis=1), 1.0, atol=1e-13)
        for k in range(Pc + 1):
            assert np.max(np.abs(I @ xc ** k - xf ** k)) < 1e-12
    assert np.allclose(interp_matrix(basis, 4, 4), np.eye(5), atol=1e-14)
    # midpoint of the linear GLL basis
    assert np.allclose(lagrange(np.array([-1.0, 1.0]), [0.0]), [[0.5, 0.5]])


def test_penalty_examples():
    for P, D, exp in _golden("penalty_examples.txt"):
        assert math.isclose(penalty_min(int(P), float(D)), float(exp), rel_tol=1e-14)


def test_c1_penalty_is_spec_definition():
    """BASELINE c1 runs "penalty mu as defined in SPEC.md": mu = 2 penalty_min(P, Delta) with
    penalty_min = P(P+1)/Delta — 160 at P = 4, Delta = 1/4.
    The oracle's operator must assemble exactly that mu from c1's penalty factor."""
    from oracle.basis import penalty_min, stability_threshold
    from workloads import get_config
    c = get_config("c1")
    delta = c.length[0] / c.ne[0]
    mu = c.penalty * stability_threshold(c.P, delta)
    assert abs(mu - 2 * penalty_min(c.P, delta)) <= 1e-12 * mu
    assert abs(mu - 160.0) <= 1e-12
