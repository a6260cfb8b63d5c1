"""O5/O6 — overlap resolution and hat weights (Table 1 :389-418,
Table 2 :524-547).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings (R5-R7):
* Overlap layers per level/direction (identical on both sides on a uniform
  grid): count the neighbour-element nodes whose face distance d (reference
  units, element width 2) satisfies d <= delta_ref (GLL) or d < delta_ref (GL),
  tolerance 1e-12, delta_ref = 2 delta_O / Delta_d; then max with the floor and
  cap at n = P+1.  FixedNodes(n_o) -> min(n_o, n).
* Reach of the weight transition (reading R6): the "subdomain boundary" of the Fig. 2 caption is
  the first neighbour node OUTSIDE the window (where the subdomain problem is Dirichlet-
  truncated): delta_ref = d_{n_o+1}, or 2 if the window covers the whole neighbour; this one
  rule serves every overlap mode.  It reproduces Table 1 rows 3, 4, 9, 13 (GPU sweep in
  profiles/), where the geometric reach 2 delta_O / Delta did not.
* Hat weight (Fig. 2 caption): xi_H = xi in the own element,
  xi -/+ 2 in the left/right neighbour; h = min(delta_ref, 1) (0 if the side has
  no overlap layer); t = (1 + h - |xi_H|) / (2 h) clipped to [0, 1];
  w = q(t) = 10 t^3 - 15 t^4 + 6 t^5: the caption fixes "piece-wise quintic"; this is the
  unique quintic with q(0) = 0, q(1) = 1 and C^2 contact at both ends (pinned by solving those
  six conditions, tests/test_oracle_schwarz.py), and Table 1 discriminates it from the
  lower-order transitions (cubic smoothstep: rows 9/13 come out 0.87/1.59 against the printed
  1.15/1.75; linear ramp: 1.06 against 1.75; the quintic: 1.147/1.752 —
  tests/test_oracle_mg.py::test_table1_rates_pin_the_quintic_transition).  What stays a reading
  (the exact definition is in the absent [Stiller2016]) is the C^2 contact itself: a C^3 septic
  smoothstep gives the same rates to 0.05, but is not "quintic".
"""
import numpy as np
from .basis import GLL, GL, face_distances

OVL_NODES, OVL_REL, OVL_MAXREL = 0, 1, 2
TOL = 1e-12


def _count(basis, P, delta_ref):
    d = face_distances(basis, P)
    if basis == GLL:
        return int(np.sum(d <= delta_ref + TOL))
    return int(np.sum(d < delta_ref - TOL))


def _first_excluded(basis, P, n_o):
    """Face distance of the first neighbour node outside the window (2: whole neighbour inside)."""
    d = face_distances(basis, P)
    return 2.0 if n_o >= P + 1 else float(d[n_o])


def resolve_overlap(mode, value, floor, basis, P, deltas):
    """Return [(n_o, delta_ref)] for the three directions at degree P."""
    n = P + 1
    out = []
    dmax = max(deltas)
    for dd in deltas:
        if mode == OVL_NODES:
            n_o = min(int(value), n)
            n_o2 = min(max(n_o, floor), n)
            out.append((n_o2, _first_excluded(basis, P, n_o2)))
            continue
        if mode == OVL_REL:
            delta_O = value * dd
        elif mode == OVL_MAXREL:
            delta_O = min(value * dmax, dd)
        else:
            raise ValueError("unknown overlap mode")
        c = min(_count(basis, P, 2.0 * delta_O / dd), n)
        c = min(max(c, floor), n)
        out.append((c, _first_excluded(basis, P, c)))
    return out


def quintic(t):
    t = np.clip(t, 0.0, 1.0)
    return t * t * t * (10.0 - 15.0 * t + 6.0 * t * t)


def hat_weight(xi_h, h):
    """w_H(xi_H) for a symmetric subdomain with transition half-width h on both sides."""
    xi_h = np.asarray(xi_h, dtype=float)
    if h <= 0.0:
        return np.where(np.abs(xi_h) <= 1.0 + TOL, 1.0, 0.0)
    return quintic((1.0 + h - np.abs(xi_h)) / (2.0 * h))


def window_1d(basis, P, n_o):
    """Window of one direction: list of (element offset, local node) and the xi_H of each node."""
    from .basis import nodes_weights
    x, _ = nodes_weights(basis, P)
    n = P + 1
    pos, xih = [], []
    for t in range(n - n_o, n):
        pos.append((-1, t)); xih.append(x[t] - 2.0)
    for i in range(n):
        pos.append((0, i)); xih.append(x[i])
    for t in range(n_o):
        pos.append((1, t)); xih.append(x[t] + 2.0)
    return pos, np.array(xih)


def weights_1d(basis, P, n_o, delta_ref):
    _, xih = window_1d(basis, P, n_o)
    h = min(delta_ref, 1.0) if n_o > 0 else 0.0
    return hat_weight(xih, h)
