"""GPU-vs-oracle parity (run on a B200 with `pytest -m gpu`), through the C ABI.

Bar (BASELINE.json north_star): relative max-norm error <= 1e-11 for the operator apply and
one V-cycle's iterate; residual-reduction factor per cycle equal to 3 significant digits.
Oracle: oracle.mf (validated against the explicit-matrix oracle.dense by the CPU suite) and
oracle.dense directly on the small grids.  Inputs: workloads (seeded, shared).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import get_config, uniform_zero_mean, uniform_vector
from workloads.configs import OverlapSpec, Config
from oracle.mf import MFHierarchy
from oracle.dense import DenseHierarchy
from oracle import mg

from tolerances import TOL, TOL_ANISO, TOL_ANISO_RES   # each bar's derivation is in tolerances.py


def _tol(name):
    return TOL_ANISO if name.startswith("c5") or name.startswith("e-aniso") else TOL


def _gpu(c):
    from paper_1612_04796_b200 import DG
    return DG(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)


def _t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda")


def _n(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _rel(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


_HCACHE = {}


def _oracle(c, dense=False):
    key = (c.name, c.ne, c.length, c.P, c.basis, c.overlap, dense)
    if key not in _HCACHE:
        cls = DenseHierarchy if dense else MFHierarchy
        _HCACHE[key] = cls(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    return _HCACHE[key]


SMALL = [("c1", None), ("c2", 3), ("c3", 3), ("c4", 3), ("c5", 3)]
FULL = ["c1", "c2", "c4", "c5"]


@pytest.mark.parametrize("name,ne", SMALL + [(n, None) for n in FULL[1:]] + [("c3", None)])
def test_apply_parity(name, ne):
    c = get_config(name, ne)
    g = _gpu(c)
    H = _oracle(c)
    u = uniform_vector(c.ndofs, 1)
    Au = _n(g.apply(_t(u)))
    ref = H.apply(H.L, u)
    assert _rel(Au, ref) <= TOL
    # every level's operator
    for l in range(H.L):
        ul = uniform_vector(H.ndofs(l), 2)
        assert _rel(_n(g.apply(_t(ul), level=l)), H.apply(l, ul)) <= TOL
    f = uniform_zero_mean(c.ndofs, 0)
    assert _rel(_n(g.residual(_t(u), _t(f))), f - ref) <= TOL


@pytest.mark.parametrize("name,ne", [("c1", None), ("c2", 3)])
def test_apply_parity_dense(name, ne):
    c = get_config(name, ne)
    g = _gpu(c)
    H = _oracle(c, dense=True)
    u = uniform_vector(c.ndofs, 1)
    assert _rel(_n(g.apply(_t(u))), H.apply(H.L, u)) <= TOL


@pytest.mark.parametrize("name,ne", SMALL)
def test_smoother_transfer_coarse_parity(name, ne):
    c = get_config(name, ne)
    g = _gpu(c)
    H = _oracle(c)
    rng = np.random.default_rng(11)
    for l in range(1, H.L + 1):
        u = rng.uniform(-1, 1, H.ndofs(l))
        f = rng.uniform(-1, 1, H.ndofs(l))
        ug = _t(u)
        g.schwarz_smooth(ug, _t(f), steps=2, level=l)
        assert _rel(_n(ug), H.smooth(l, u, f, 2)) <= _tol(name), l
        uc = rng.uniform(-1, 1, H.ndofs(l - 1))
        ug = _t(u)
        g.prolongate_add(_t(uc), ug, l)
        assert _rel(_n(ug), u + H.prolong(l, uc)) <= TOL
        assert _rel(_n(g.restrict(_t(f), l)), H.restrict(l, f)) <= TOL
    f0 = rng.uniform(-1, 1, H.ndofs(0))
    assert _rel(_n(g.coarse_solve(_t(f0))), H.coarse(f0)) <= TOL


@pytest.mark.parametrize("name,ne", SMALL + [(n, None) for n in FULL[1:]])
def test_vcycle_parity(name, ne):
    c = get_config(name, ne)
    g = _gpu(c)
    H = _oracle(c)
    f = uniform_zero_mean(c.ndofs, 0)
    u = np.zeros(c.ndofs)
    ug, fg = _t(u), _t(f)
    # Two cycles everywhere except full-size c5, whose plain V-cycle diverges after the first
    # (||r||/||r0|| = 0.17, 1.2, 9.8 for cycles 1-3; the paper runs it only inside CG for high
    # aspect ratios): a divergent iteration amplifies the round-off of cycle 1 (GPU and oracle
    # then differ by 8e-10 after cycle 2, scripts/c5_gap_probe.py), so that case stops at one.
    for k in range(1 if (name == "c5" and ne is None) else 2):
        g.pmg_vcycle(ug, fg)
        u = mg.vcycle(H, u, f)
        assert _rel(_n(ug), u) <= _tol(name), k
        # conditioning-insensitive check: the two iterates have the same residual to TOL of
        # ||f|| (c5: TOL_ANISO_RES, 5x the dense-vs-FDM oracle floor; tolerances.py)
        dr = H.apply(H.L, _n(ug) - u)
        assert np.max(np.abs(dr)) <= (TOL if _tol(name) == TOL else TOL_ANISO_RES) * np.max(np.abs(f)), k


def test_vcycle_parity_c3_full():
    test_vcycle_parity("c3", None)


@pytest.mark.parametrize("name,ne,cycles", [("c1", None, 12), ("c2", None, 10), ("c4", 3, 6), ("c3", 4, 6),
                                             ("c3", None, 5), ("c4", None, 5)])
def test_rate_per_cycle_three_digits(name, ne, cycles):
    c = get_config(name, ne)
    g = _gpu(c)
    H = _oracle(c)
    if c.rhs == "uniform":
        f = uniform_zero_mean(c.ndofs, 0)
        fg = _t(f)
    else:                         # each side assembles its own sin-product RHS (c2)
        f = _sin_rhs_oracle(c)
        fg = g.rhs_sin(3.0, 1.0, 1.0, 1.0)
    ug = torch.zeros_like(fg)
    u = np.zeros(c.ndofs)
    r_g, r_o = [np.sqrt(g.dot(fg, fg))], [np.linalg.norm(f)]
    for k in range(cycles):
        g.pmg_vcycle(ug, fg)
        u = mg.vcycle(H, u, f)
        res = g.residual(ug, fg)
        r_g.append(np.sqrt(g.dot(res, res)))
        r_o.append(mg.residual_norm(H, u, f))
        if r_o[-1] / r_o[0] < 1e-9:
            break
    rho_g = np.array(r_g[1:]) / np.array(r_g[:-1])
    rho_o = np.array(r_o[1:]) / np.array(r_o[:-1])
    assert np.all(np.abs(rho_g - rho_o) <= 5e-4 * np.abs(rho_o)), (rho_g, rho_o)


def _sin_rhs_oracle(c):
    from oracle.dense import mass_diag, node_coords
    X, Y, Z = node_coords(c.ne, c.length, c.P, c.basis)
    b = mass_diag(c.ne, c.length, c.P, c.basis) * 3 * np.sin(X) * np.sin(Y) * np.sin(Z)
    return b - b.mean()


def test_rhs_sin_matches_oracle():
    c = get_config("c2")
    g = _gpu(c)
    b = _sin_rhs_oracle(c)
    assert np.max(np.abs(_n(g.rhs_sin(3.0, 1.0, 1.0, 1.0)) - b)) <= TOL * np.max(np.abs(b))


@pytest.mark.parametrize("ne", [3, None])
def test_pcg_parity_c5(ne):
    c = get_config("c5", ne)
    g = _gpu(c)
    H = _oracle(c)
    f = uniform_zero_mean(c.ndofs, 0)
    ug = torch.zeros(c.ndofs, dtype=torch.float64, device="cuda")
    _, hist_g, ok = g.pcg_solve(ug, _t(f), rtol=1e-10, maxit=200)
    u, hist_o = mg.pcg(H, f, rtol=1e-10, maxit=200)
    assert ok and len(hist_g) == len(hist_o)
    # relative residual histories agree to 3 significant digits while above round-off
    sel = np.array(hist_o) / hist_o[0] >= 1e-9
    assert np.all(np.abs(hist_g[sel] - np.array(hist_o)[sel]) <= 5e-4 * np.array(hist_o)[sel])
    assert _rel(_n(ug), u) <= 1e-8      # final iterates (converged to 1e-10 relative residual)


# ---- edge cases: minimum grid, P=2, no overlap, full-neighbour overlap, anisotropy
EDGE = [
    Config("e-min", (3, 3, 3), (1.0, 1.0, 1.0), 2, 0, OverlapSpec(0, 1, 0)),
    Config("e-noovl", (3, 4, 5), (1.0, 1.2, 1.5), 4, 1, OverlapSpec(0, 0, 0)),
    Config("e-full", (3, 3, 4), (1.0, 1.0, 1.3), 4, 0, OverlapSpec(0, 5, 0)),
    Config("e-gl-half", (4, 3, 3), (2.0, 1.0, 1.0), 8, 1, OverlapSpec(1, 0.5, 0)),
    Config("e-aniso", (5, 3, 4), (20.0, 1.0, 0.5), 4, 1, OverlapSpec(2, 0.08, 1)),
]


@pytest.mark.parametrize("c", EDGE, ids=[e.name for e in EDGE])
def test_edge_cases(c):
    g = _gpu(c)
    H = MFHierarchy(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    u = uniform_vector(c.ndofs, 1)
    assert _rel(_n(g.apply(_t(u))), H.apply(H.L, u)) <= TOL
    f = uniform_zero_mean(c.ndofs, 0)
    ug = torch.zeros(c.ndofs, dtype=torch.float64, device="cuda")
    g.pmg_vcycle(ug, _t(f))
    assert _rel(_n(ug), mg.vcycle(H, np.zeros_like(f), f)) <= _tol(c.name)


def test_determinism_bitwise():
    c = get_config("c2", 4)
    g = _gpu(c)
    f = _t(uniform_zero_mean(c.ndofs, 0))
    outs = []
    for _ in range(2):
        u = torch.zeros_like(f)
        for _ in range(2):
            g.pmg_vcycle(u, f)
        outs.append(_n(u))
    assert np.array_equal(outs[0], outs[1])


def test_errors_fail_loudly():
    from paper_1612_04796_b200 import DG, PMGError
    g = DG((4, 4, 4), (1, 1, 1), 4, 0, overlap=None)
    u = torch.zeros(g.ndofs(), dtype=torch.float64, device="cuda")
    with pytest.raises(PMGError):
        g.pmg_vcycle(u, u)                  # no Schwarz setup / aliased
    with pytest.raises(PMGError):
        g.apply(u, out=u)                   # aliased


# ---- NEXT rows: variable V-cycle (Table 2) and the large-window global path
def test_variable_vcycle_schedule():
    c = get_config("c2", 3)
    g = _gpu(c)
    H = _oracle(c)
    nu = [0] + [3 ** (H.L - l) for l in range(1, H.L + 1)]      # (1,1) x 3^(L-l)
    g.set_schedule(nu, nu)
    f = uniform_zero_mean(c.ndofs, 0)
    ug = torch.zeros(c.ndofs, dtype=torch.float64, device="cuda")
    g.pmg_vcycle(ug, _t(f))
    assert _rel(_n(ug), mg.vcycle(H, np.zeros_like(f), f, growth=3)) <= TOL


BIG = [
    Config("e-gll05-p16", (3, 3, 3), (1.0, 1.0, 1.0), 16, 0, OverlapSpec(1, 0.5, 0)),     # m = 35
    Config("e-full-p16", (3, 3, 4), (1.0, 1.0, 1.3), 16, 0, OverlapSpec(0, 17, 0)),      # m = 51
]


def test_very_large_windows_scalar_path():
    """Windows beyond the global line-GEMM path (m > 80: P = 32 with n_o = 25 layers, m = 83) run the
    scalar FP64 kernel k_fdm; one top-level Schwarz step against the oracle."""
    c = Config("e-p32-no25", (4, 3, 3), (1.0, 1.0, 1.0), 32, 0, OverlapSpec(0, 25, 0))
    g = _gpu(c)
    assert g.level_overlap(g.L)[1] == [83, 83, 83]
    H = MFHierarchy(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    f = uniform_zero_mean(c.ndofs, 0)
    u = uniform_vector(c.ndofs, 1)
    ug = _t(u)
    g.schwarz_smooth(ug, _t(f), steps=1)
    assert _rel(_n(ug), H.smooth(H.L, u, f, 1)) <= TOL


@pytest.mark.parametrize("c", BIG, ids=[e.name for e in BIG])
def test_large_windows_global_path(c):
    g = _gpu(c)
    H = MFHierarchy(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    f = uniform_zero_mean(c.ndofs, 0)
    u = uniform_vector(c.ndofs, 1)
    ug = _t(u)
    g.schwarz_smooth(ug, _t(f), steps=1)
    assert _rel(_n(ug), H.smooth(H.L, u, f, 1)) <= TOL
    ug = torch.zeros(c.ndofs, dtype=torch.float64, device="cuda")
    g.pmg_vcycle(ug, _t(f))
    assert _rel(_n(ug), mg.vcycle(H, np.zeros_like(f), f)) <= TOL


def _table1():
    import os
    rows = {}
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "table1_rates.txt")):
        line = line.split("#")[0].split()
        if line:
            rows[int(line[0])] = (line[1], line[2], OverlapSpec(int(line[3]), float(line[4]), int(line[5])),
                                  [float(x) for x in line[6:10]])
    return rows


@pytest.mark.parametrize("row,P", [(1, 16), (1, 32), (7, 16), (7, 32), (2, 32), (8, 32),
                                   (3, 8), (3, 16), (4, 8), (4, 16), (9, 8), (9, 16), (10, 8), (10, 16),
                                   (13, 8), (13, 16), (14, 8), (14, 16)])
def test_table1_rates_at_paper_scale(row, P):
    """The GPU (parity-pinned to the oracle) reproduces Table 1 at the paper's own grids: -lg rho
    within 0.06 of the printed value (paper protocol: random guess in [-1,1], RHS
    M 3 sin x sin y sin z, iterate to 1e-10; Table 1 :401-415).  Rows 3, 4, 9,
    10, 13, 14 (relative overlaps) have window nodes inside the weight transition band, so they
    pin the hat-weight reach of reading R6; rows 1, 2, 7, 8 (one node of overlap) pin the
    operator, the transfers and the solver."""
    import math
    basis, solver, ov, paper = _table1()[row]
    from paper_1612_04796_b200 import DG
    ne = 128 // P
    L2 = 2 * math.pi
    g = DG((ne, ne, ne), (L2, L2, L2), P, 0 if basis == "GLL" else 1, 2.0, ov)
    f = g.rhs_sin(3.0, 1.0, 1.0, 1.0)
    u = _t(uniform_vector(g.ndofs(), 3))
    if solver == "MG-CG":
        _, hist, ok = g.pcg_solve(u, f, rtol=1e-10, maxit=80)
        assert ok
    else:
        r = g.residual(u, f)
        hist = [math.sqrt(g.dot(r, r))]
        for _ in range(80):
            g.pmg_vcycle(u, f)
            r = g.residual(u, f)
            hist.append(math.sqrt(g.dot(r, r)))
            if hist[-1] <= 1e-10 * hist[0]:
                break
    lg = -math.log10((hist[-1] / hist[0]) ** (1.0 / (len(hist) - 1)))
    want = paper[[4, 8, 16, 32].index(P)]
    assert abs(lg - want) <= 0.06, (lg, want)


def test_c2_manufactured_solution_accuracy():
    """NEXT row f4 / BASELINE c2: V(1,1) cycles on the GPU until ||r||/||r0|| <= 1e-10 for
    f = M 3 sin x sin y sin z; the discrete solution approximates u = sin x sin y sin z to
    O(h^{P+1}) (P = 8, h = pi/4: nodal error well below 1e-6), and the per-cycle reduction is
    the paper's row-13 regime (-lg rho = 1.75 at P = 8)."""
    import math
    from oracle.dense import node_coords
    c = get_config("c2")
    g = _gpu(c)
    f = g.rhs_sin(3.0, 1.0, 1.0, 1.0)
    u = torch.zeros_like(f)
    r0 = math.sqrt(g.dot(f, f))
    hist = [r0]
    for _ in range(30):
        g.pmg_vcycle(u, f)
        r = g.residual(u, f)
        hist.append(math.sqrt(g.dot(r, r)))
        if hist[-1] <= 1e-10 * r0:
            break
    assert hist[-1] <= 1e-10 * r0
    lg = -math.log10((hist[-1] / hist[0]) ** (1.0 / (len(hist) - 1)))
    assert lg > 1.0, lg          # zero initial guess + smooth RHS on 8^3 (paper: 16^3, random guess)
    X, Y, Z = node_coords(c.ne, c.length, c.P, c.basis)
    ue = np.sin(X) * np.sin(Y) * np.sin(Z)
    err = _n(u) - ue
    err -= err.mean()
    assert np.max(np.abs(err)) < 1e-6, np.max(np.abs(err))


@pytest.mark.parametrize("name,ne", [("c1", None), ("c3", 4)])
def test_colored_scatter_matches_oracle(name, ne):
    """dg_set_colored(1): the Schwarz correction added colour by colour straight into u."""
    c = get_config(name, ne)
    g = _gpu(c)
    g.set_colored(True)
    H = _oracle(c)
    f = uniform_zero_mean(c.ndofs, 0)
    ug = torch.zeros(c.ndofs, dtype=torch.float64, device="cuda")
    u = np.zeros(c.ndofs)
    for _ in range(2):
        g.pmg_vcycle(ug, _t(f))
        u = mg.vcycle(H, u, f)
        assert _rel(_n(ug), u) <= TOL


@pytest.mark.parametrize("name,ne", [("c1", None), ("c2", 3), ("c3", 3), ("c4", 3)])
def test_pcg_parity_all_configs(name, ne):
    """MG-CG (Table 1 even rows) on every config family: residual histories to 3 digits."""
    c = get_config(name, ne)
    g = _gpu(c)
    H = _oracle(c)
    f = uniform_zero_mean(c.ndofs, 0)
    ug = torch.zeros(c.ndofs, dtype=torch.float64, device="cuda")
    _, hist_g, ok = g.pcg_solve(ug, _t(f), rtol=1e-10, maxit=80)
    u, hist_o = mg.pcg(H, f, rtol=1e-10, maxit=80)
    assert ok and len(hist_g) == len(hist_o)
    sel = np.array(hist_o) / hist_o[0] >= 1e-9
    assert np.all(np.abs(hist_g[sel] - np.array(hist_o)[sel]) <= 5e-4 * np.array(hist_o)[sel])
    assert _rel(_n(ug), u) <= 1e-9


def test_vector_helpers_and_coarse_at_c3_size():
    c = get_config("c3")
    g = _gpu(c)
    H = _oracle(c)
    x = uniform_vector(c.ndofs, 5)
    y = uniform_vector(c.ndofs, 6)
    assert abs(g.dot(_t(x), _t(y)) - float(x @ y)) <= 1e-12 * np.abs(x).dot(np.abs(y))
    xp = _t(x)
    g.project_mean(xp)
    assert _rel(_n(xp), x - x.mean()) <= TOL
    f0 = uniform_vector(H.ndofs(0), 7)         # 32^3 coarse grid (fused 5-kernel path)
    assert _rel(_n(g.coarse_solve(_t(f0))), H.coarse(f0)) <= TOL


@pytest.mark.parametrize("ne,length", [((6, 5, 7), (1.0, 1.0, 1.0)), ((16, 4, 9), (3.0, 1.0, 2.0)),
                                       ((5, 6, 16), (1.0, 2.0, 1.0)), ((8, 8, 8), (1.0, 1.0, 1.0)),
                                       ((16, 12, 14), (1.0, 1.0, 1.0)), ((9, 16, 11), (2.0, 1.0, 1.0))])
def test_coarse_cluster_ragged(ne, length):
    """Coarse pseudo-inverse (Alg. 1 l.295) on the one-cluster path with non-cubic grids whose
    z extent does not divide evenly over the 8 CTAs (G_z = 14, 18, 32; some CTAs own no plane),
    and on c2's 16^3 grid; the last two grids (N_0 > 8192) take the three-launch plane path."""
    c = Config("coarse", ne, length, 2, 0, OverlapSpec(0, 1, 0))
    g = _gpu(c)
    H = _oracle(c)
    f0 = uniform_vector(H.ndofs(0), 11)
    assert _rel(_n(g.coarse_solve(_t(f0))), H.coarse(f0)) <= TOL


def test_single_level_hierarchy_p2():
    """P = 2: one smoothing level above the P = 1 coarse level (L = 1)."""
    c = Config("p2", (4, 4, 4), (1.0, 1.0, 1.0), 2, 1, OverlapSpec(1, 0.5, 0))
    g = _gpu(c)
    H = MFHierarchy(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    f = uniform_zero_mean(c.ndofs, 0)
    ug = torch.zeros(c.ndofs, dtype=torch.float64, device="cuda")
    u = np.zeros(c.ndofs)
    for _ in range(3):
        g.pmg_vcycle(ug, _t(f))
        u = mg.vcycle(H, u, f)
    assert _rel(_n(ug), u) <= TOL


def test_workspace_and_state_errors():
    from paper_1612_04796_b200 import DG, PMGError
    from paper_1612_04796_b200.binding import lib
    import ctypes as C
    g = DG((4, 4, 4), (1, 1, 1), 4, 0, overlap=OverlapSpec(0, 1, 0), bind=False)
    small = torch.empty(1024, dtype=torch.uint8, device="cuda")
    rc = lib.dg_bind_workspace(g._c, C.c_void_p(small.data_ptr()), 1024, None)
    assert rc == 5                                   # PMG_EWORKSPACE
    u = torch.zeros(g.ndofs(), dtype=torch.float64, device="cuda")
    with pytest.raises(PMGError):
        g.apply(u)                                   # workspace not bound -> PMG_ESTATE


# ---- ragged (non-cubic) element grids with the benchmark window shapes: the compile-time
# Schwarz kernels (23^3, 13^3, 11x27x27, ...), the n = 17 apply column table and the 3-CTA
# prolongation on grids whose element counts per direction differ (periodic wrap per axis)
RAGGED = [("c3", (3, 4, 3)), ("c5", (4, 3, 5)), ("c2", (5, 3, 4))]


@pytest.mark.parametrize("name,ne", RAGGED, ids=[r[0] for r in RAGGED])
def test_ragged_grids_benchmark_shapes(name, ne):
    c = get_config(name, ne)
    g = _gpu(c)
    H = _oracle(c)
    u = uniform_vector(c.ndofs, 1)
    assert _rel(_n(g.apply(_t(u))), H.apply(H.L, u)) <= TOL
    f = uniform_zero_mean(c.ndofs, 0)
    ug = torch.zeros(c.ndofs, dtype=torch.float64, device="cuda")
    uo = np.zeros_like(f)
    for _ in range(2):
        g.pmg_vcycle(ug, _t(f))
        uo = mg.vcycle(H, uo, f)
    assert _rel(_n(ug), uo) <= _tol(c.name)


@pytest.mark.parametrize("name,ne", [("c5", 3), ("c2", 3), ("c1", None)])
def test_pcg_graph_equals_host_loop(name, ne):
    """pcg_solve as one CUDA-graph launch (conditional WHILE/IF nodes, device-side convergence
    test) gives the host-driven loop's iterates and residual history bit for bit."""
    c = get_config(name, ne)
    out = []
    for graphs in (True, False):
        g = _gpu(c)
        g.set_graphs(graphs)
        f = _t(uniform_zero_mean(c.ndofs, 0))
        u = torch.zeros_like(f)
        _, hist, ok = g.pcg_solve(u, f, rtol=1e-10, maxit=200)
        assert ok
        out.append((_n(u), np.array(hist)))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    # a solve that hits maxit reports PMG_EMAXIT through the graph path too
    g = _gpu(c)
    u = torch.zeros(c.ndofs, dtype=torch.float64, device="cuda")
    _, hist, ok = g.pcg_solve(u, _t(uniform_zero_mean(c.ndofs, 0)), rtol=1e-14, maxit=3)
    assert not ok and len(hist) == 4


@pytest.mark.parametrize("basis,P,k", [(0, 2, 6), (1, 2, 6), (0, 4, 4), (1, 4, 4)])
def test_gpu_convergence_order(basis, P, k):
    """NEXT row f4: the GPU solve of A u = M 3 sin x sin y sin z converges to u = sin x sin y sin z
    at O(h^{P+1}) under mesh refinement k^3 -> (2k)^3 (north_star), same bounds
    as the oracle's own CPU pin (test_oracle_operator.test_convergence_order)."""
    import math
    from oracle.dense import node_coords
    from oracle.dense import mass_diag
    errs = []
    for kk in (k, 2 * k):
        c = Config("order", (kk, kk, kk), (2 * math.pi,) * 3, P, basis, OverlapSpec(1, 0.09, 1))
        g = _gpu(c)
        f = g.rhs_sin(3.0, 1.0, 1.0, 1.0)
        u = torch.zeros_like(f)
        _, hist, ok = g.pcg_solve(u, f, rtol=1e-13, maxit=80)
        assert ok
        X, Y, Z = node_coords(c.ne, c.length, c.P, c.basis)
        M = mass_diag(c.ne, c.length, c.P, c.basis)
        err = _n(u) - np.sin(X) * np.sin(Y) * np.sin(Z)
        err -= np.sum(M * err) / np.sum(M)
        errs.append(math.sqrt(np.sum(M * err * err)))
    order = math.log2(errs[0] / errs[1])
    assert P + 0.75 <= order <= P + 2.25, (order, errs)


@pytest.mark.parametrize("name,ne", [("c1", None), ("c2", 4), ("c3", 3), ("c5", 4)])
def test_slab_decomposition_single_rank_equals_plain(name, ne):
    """NEXT row f3: the element-slab path (SlabDG: local mesh = owned layers +
    two ghost layers, halo exchanges of u, r and the window buffer inside every Schwarz step,
    gathered coarse solve) with ONE rank — the ghost layers are then the rank's own periodic
    images — must reproduce the plain single-GPU V-cycles on the owned layers, and the oracle."""
    from paper_1612_04796_b200 import SlabDG
    c = get_config(name, ne)
    g = _gpu(c)
    sd = SlabDG(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    assert sd.world == 1 and sd.local_ne[2] == c.ne[2] + 2
    f = uniform_zero_mean(c.ndofs, 0)
    fg = _t(f)
    u_plain = torch.zeros_like(fg)
    fl = sd.scatter_global(fg)
    ul = torch.zeros_like(fl)
    H = _oracle(c)
    u_ref = np.zeros_like(f)
    for _ in range(2):
        g.pmg_vcycle(u_plain, fg)
        sd.vcycle(ul, fl)
        u_ref = mg.vcycle(H, u_ref, f)
        got = _n(sd.gather_global(ul))
        assert _rel(got, _n(u_plain)) <= 1e-12
        assert _rel(got, u_ref) <= _tol(name)
    assert sd.exchanges > 0
    # residual norm through the owned-range dot equals the plain one
    r_plain = g.residual(u_plain, fg)
    r_slab = sd.residual(ul, fl)
    assert abs(sd.dot(r_slab, r_slab) - g.dot(r_plain, r_plain)) <= 1e-10 * g.dot(r_plain, r_plain)


@pytest.mark.parametrize("name,ne", [("c5", 4), ("c2", 4)])
def test_slab_pcg_single_rank_equals_plain(name, ne):
    """Slab form of the inexact PCG (all-reduced scalars, dg_axpby updates) with
    one rank: same iteration count and residual history as the library's pcg_solve, same solution."""
    from paper_1612_04796_b200 import SlabDG
    c = get_config(name, ne)
    g = _gpu(c)
    sd = SlabDG(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    f = uniform_zero_mean(c.ndofs, 0)
    fg = _t(f)
    u_plain = torch.zeros_like(fg)
    _, h_plain, ok = g.pcg_solve(u_plain, fg, rtol=1e-10, maxit=300)
    assert ok
    fl = sd.scatter_global(fg)
    ul = torch.zeros_like(fl)
    _, h_slab, ok2 = sd.pcg_solve(ul, fl, rtol=1e-10, maxit=300)
    assert ok2 and len(h_slab) == len(h_plain)
    assert np.allclose(h_slab, h_plain, rtol=1e-6)
    assert _rel(_n(sd.gather_global(ul)), _n(u_plain)) <= 1e-8
