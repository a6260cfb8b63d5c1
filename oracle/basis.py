"""O1 — 1D nodal bases on GL / GLL points (§2 Eq. 5).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* GL nodes  = roots of the Legendre polynomial P_{P+1}
* GLL nodes = {-1, +1} U roots of P'_P
* Lagrange basis phi_j(x) = prod_{k != j} (x - xi_k)/(xi_j - xi_k), evaluated
  by that product directly; phi'_j by the product rule written out.
"""
from functools import lru_cache
import numpy as np
from numpy.polynomial import legendre as npleg

GLL, GL = 0, 1


def _legendre_coeffs(k):
    c = np.zeros(k + 1)
    c[k] = 1.0
    return c


@lru_cache(maxsize=None)
def nodes_weights(basis, P):
    """Nodes (ascending) and quadrature weights on [-1, 1] for degree P."""
    if P < 1:
        raise ValueError("P must be >= 1 (SPEC.md:97)")
    if basis == GL:
        x, w = npleg.leggauss(P + 1)        # Gauss-Legendre rule with P+1 points
        return np.array(x), np.array(w)
    if basis != GLL:
        raise ValueError("basis must be GLL (0) or GL (1)")
    cP = _legendre_coeffs(P)
    d1 = npleg.legder(cP)
    d2 = npleg.legder(cP, 2)
    if P == 1:
        inner = np.array([])
    else:
        inner = np.sort(np.real(npleg.legroots(d1)))
        for _ in range(8):                   # Newton polish of the roots of P'_P
            inner = inner - npleg.legval(inner, d1) / npleg.legval(inner, d2)
    x = np.concatenate([[-1.0], inner, [1.0]])
    # Lobatto weights w_i = 2 / (P (P+1) P_P(x_i)^2)
    w = 2.0 / (P * (P + 1) * npleg.legval(x, cP) ** 2)
    return x, w


def lagrange(nodes, x):
    """Matrix [len(x), n]: phi_j(x_q) by the Lagrange product formula."""
    nodes = np.asarray(nodes, dtype=float)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    n = len(nodes)
    out = np.ones((len(x), n))
    for j in range(n):
        for k in range(n):
            if k != j:
                out[:, j] *= (x - nodes[k]) / (nodes[j] - nodes[k])
    return out


def lagrange_deriv(nodes, x):
    """Matrix [len(x), n]: phi_j'(x_q) = sum_{m != j} 1/(xi_j - xi_m) prod_{k != j,m} (x - xi_k)/(xi_j - xi_k)."""
    nodes = np.asarray(nodes, dtype=float)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    n = len(nodes)
    out = np.zeros((len(x), n))
    for j in range(n):
        for m in range(n):
            if m == j:
                continue
            prod = np.full(len(x), 1.0 / (nodes[j] - nodes[m]))
            for k in range(n):
                if k != j and k != m:
                    prod = prod * (x - nodes[k]) / (nodes[j] - nodes[k])
            out[:, j] += prod
    return out


@lru_cache(maxsize=None)
def basis_data(basis, P):
    """Everything the assembly needs: nodes, weights, D[q, j] = phi_j'(xi_q),
    traces phi(-1), phi(+1), phi'(-1), phi'(+1) (each length n)."""
    x, w = nodes_weights(basis, P)
    D = lagrange_deriv(x, x)
    ends = np.array([-1.0, 1.0])
    val = lagrange(x, ends)
    der = lagrange_deriv(x, ends)
    return dict(x=x, w=w, D=D, phi_m=val[0], phi_p=val[1], dphi_m=der[0], dphi_p=der[1])


def interp_matrix(basis, P_from, P_to):
    """Embedded interpolation I (§3.2): I[i, j] = phi_j^{(P_from)}(xi_i^{(P_to)})."""
    xf, _ = nodes_weights(basis, P_from)
    xt, _ = nodes_weights(basis, P_to)
    return lagrange(xf, xt)


def face_distances(basis, P):
    """Reference-unit distances (element width = 2) of the nodes from the face at xi = -1,
    ascending."""
    x, _ = nodes_weights(basis, P)
    return x + 1.0


def penalty_min(P, delta):
    """The printed example mu_min = P(P+1)/Delta."""
    return P * (P + 1) / delta


def stability_threshold(P, delta):
    """Coercivity threshold of this SIPG normalisation (reading R2): the smallest mu for
    which the periodic 1D IP matrix is positive semi-definite is P(P+1)/(2 Delta) -- half the
    printed example; PAPER.md:331-333 defines mu_min as "the stability threshold", so the paper's
    mu = 2 mu_min is mu = 2 * stability_threshold.  Pinned by tests/test_oracle_operator.py
    (bisection on the explicit 1D matrix) and by Table 1 rows 1 and 7 (profiles/)."""
    return P * (P + 1) / (2.0 * delta)
