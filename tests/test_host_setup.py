"""CPU tests of the product's C++ host setup (through the C ABI, no GPU) against the oracle,
plus the ABI surface: the library loads and exports every symbol include/pmg_dg.h declares."""
import os
import re
import numpy as np
import pytest

from workloads import CONFIGS, get_config
from oracle.basis import basis_data, interp_matrix, nodes_weights
from oracle.mf import assemble_1d, restricted_eig
from oracle.overlap import resolve_overlap, weights_1d

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_abi_exports_every_declared_symbol():
    import ctypes
    from paper_1612_04796_b200.binding import LIB_PATH, EXPORTED
    hdr = open(os.path.join(ROOT, "include", "pmg_dg.h")).read()
    declared = set(re.findall(r"^\s*(?:int|long long|size_t|const char \*|void)\s*\*?\s*(\w+)\(", hdr, re.M))
    assert len(declared) >= 20
    so = ctypes.CDLL(LIB_PATH)
    for name in declared:
        assert hasattr(so, name), name
    assert declared == set(EXPORTED)


def test_setup_rejects_bad_arguments():
    from paper_1612_04796_b200 import DG, PMGError
    for args in [((2, 4, 4), (1, 1, 1), 4, 0), ((4, 4, 4), (1, 1, 1), 3, 0), ((4, 4, 4), (1, 1, 1), 1, 0),
                 ((4, 4, 4), (1, -1, 1), 4, 0), ((4, 4, 4), (1, 1, 1), 4, 7), ((4, 4, 4), (1, 1, 1), 64, 0)]:
        with pytest.raises(PMGError):
            DG(*args, bind=False)
    from workloads.configs import OverlapSpec
    with pytest.raises(PMGError):
        DG((4, 4, 4), (1, 1, 1), 4, 0, overlap=OverlapSpec(1, 1.5, 0), bind=False)


@pytest.mark.parametrize("name", list(CONFIGS))
def test_tables_match_oracle(name):
    from paper_1612_04796_b200 import DG
    c = get_config(name)
    g = DG(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap, bind=False)
    deltas = [c.length[d] / c.ne[d] for d in range(3)]
    for l in range(g.L + 1):
        P = 2 ** l
        n = P + 1
        x, w = nodes_weights(c.basis, P)
        assert np.allclose(g.table(l, 0, 7), x, atol=1e-15, rtol=0)
        if l >= 1:
            assert np.allclose(g.table(l, 0, 6).reshape(n, P // 2 + 1), interp_matrix(c.basis, P // 2, P),
                               atol=2e-14, rtol=0)
            res = resolve_overlap(c.overlap.mode, c.overlap.value, c.overlap.floor, c.basis, P, deltas)
            no, m = g.level_overlap(l)
            assert no == [r[0] for r in res]
        for d in range(3):
            L1, M1 = assemble_1d(c.basis, P, c.ne[d], deltas[d], c.penalty)
            assert np.allclose(g.table(l, d, 0), M1[:n], rtol=1e-14, atol=0)
            Dg = g.table(l, d, 1).reshape(n, n)
            assert np.max(np.abs(Dg - L1[n:2 * n, n:2 * n])) < 1e-12 * np.max(np.abs(L1))
            if l >= 1:
                no = res[d][0]
                win = np.arange(n - no, 2 * n + no)
                lam_o, S_o = restricted_eig(L1[np.ix_(win, win)], M1[win])
                m = len(win)
                lam = g.table(l, d, 4)
                S = g.table(l, d, 3).reshape(m, m)
                # modes come as [even ascending, odd ascending] (exact-parity eigensolver)
                assert np.allclose(np.sort(lam), np.sort(lam_o), rtol=1e-13, atol=0)
                H = m // 2
                R = S[::-1, :]                      # reflection a -> m-1-a
                assert np.array_equal(R[:, :H + 1], S[:, :H + 1])      # even modes, bit-exact
                assert np.array_equal(R[:, H + 1:], -S[:, H + 1:])     # odd modes, bit-exact
                assert np.all(np.diff(lam[:H + 1]) >= 0) and np.all(np.diff(lam[H + 1:]) >= 0)
                # sign-invariant comparison: the inverse S Lambda^-1 S^T
                inv = (S / lam) @ S.T
                inv_o = (S_o / lam_o) @ S_o.T
                assert np.max(np.abs(inv - inv_o)) < 1e-13 * np.max(np.abs(inv_o))
                assert np.max(np.abs(S.T @ (M1[win][:, None] * S) - np.eye(m))) < 1e-13
                assert np.allclose(g.table(l, d, 5), weights_1d(c.basis, P, res[d][0], res[d][1]),
                                   atol=1e-15, rtol=0)


def test_colmap17_table_is_a_conflict_free_permutation():
    """csrc/colmap17.cuh (the n = 17 apply's tile order) equals what scripts/gen_colmap17.py
    builds: a permutation of the 289 line columns in 36 full tiles (+ one single-column tile)
    whose B-load and C-store bank residues are distinct per half-warp (the generator's check)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen_colmap17", os.path.join(ROOT, "scripts", "gen_colmap17.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    tab = gen.build()
    gen.check(tab)
    hdr = open(os.path.join(ROOT, "paper_1612_04796_b200", "csrc", "colmap17.cuh")).read()
    body = re.search(r"kColMap17\[(\d+)\] = \{([^}]*)\}", hdr)
    assert int(body.group(1)) == len(tab) == 296
    assert [int(x) for x in body.group(2).split(",")] == tab
    assert sorted(tab[:289]) == list(range(289)) and set(tab[289:]) == {tab[288]}


def test_binding_rejects_wrong_vectors_before_the_abi():
    """The binding checks every vector against the ABI contract (CUDA, float64, contiguous, the
    level's DOF count) before a pointer crosses into the C library (no GPU needed: it raises first)."""
    import pytest
    import torch
    from paper_1612_04796_b200 import DG
    from workloads.configs import OverlapSpec
    g = DG((3, 3, 3), (1.0, 1.0, 1.0), 2, 0, overlap=OverlapSpec(0, 1, 0), bind=False)
    n = g.ndofs()
    with pytest.raises(ValueError):
        g.apply(torch.zeros(n, dtype=torch.float64))                        # host tensor
    with pytest.raises((ValueError, TypeError)):
        g.pmg_vcycle(torch.zeros(n, dtype=torch.float32), torch.zeros(n))   # wrong dtype / device
    with pytest.raises(ValueError):
        g.set_schedule([1, 1], [1, 1, 1])                                   # L + 1 = 2 entries each
    g.close()
