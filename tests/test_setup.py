"""Host setup (assembly, transfers, pieces, FD data) pinned to the reference.

The golden fixtures (tests/golden/*.npz, tools/make_golden.py) were produced by
running the reference igamg package; the product's own setup must reproduce
its hierarchy sizes exactly and its operators / right-hand sides to 1e-13.
When /root/reference is importable (this container) the matrices themselves
are compared directly as well.
"""

import os
import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC, SMALL_CASES, get_setup, load_golden


@pytest.mark.parametrize("golden,cfg,kw", SMALL_CASES + [("cfg2", "cfg2", {}), ("cfg3", "cfg3", {})])
def test_setup_fingerprints(golden, cfg, kw):
    g = load_golden(golden)
    pr, setup, f = get_setup(cfg, **kw)
    L = setup.finest
    assert np.array_equal(g["fp_n"], [setup.A[l].shape[0] for l in range(L + 1)])
    assert np.array_equal(g["fp_nnz"], [setup.A[l].nnz for l in range(L + 1)])
    assert np.array_equal(g["fp_p_nnz"], [0] + [setup.P[l].nnz for l in range(1, L + 1)])
    fro = np.array([np.sqrt((setup.A[l].data ** 2).sum()) for l in range(L + 1)])
    assert np.allclose(fro, g["fp_fro"], rtol=1e-13, atol=0)
    v = np.random.default_rng(0).standard_normal(setup.n_dofs)
    Av = setup.A[L] @ v
    assert np.abs(Av - g["fp_Av"]).max() <= 1e-13 * np.abs(g["fp_Av"]).max()
    assert np.abs(f - g["f"]).max() <= 1e-13 * np.abs(g["f"]).max()


def test_piece_partition_and_kinds():
    pr, setup, f = get_setup("cfg2", levels=3)
    scms = setup.smoother[3].scms
    deco = scms.decomposition
    deco.validate_partition()
    kinds = [p.kind for p in deco.pieces]
    assert kinds.count("interior") == 4 and kinds.count("edge") == 4 and kinds.count("vertex") == 1
    pr5, setup5, _ = get_setup("cfg5", levels=1)
    kinds5 = [p.kind for p in setup5.smoother[1].scms.decomposition.pieces]
    assert (kinds5.count("interior"), kinds5.count("face"), kinds5.count("edge"), kinds5.count("vertex")) == (8, 12, 6, 1)


@pytest.mark.parametrize("cfg,kw", [("cfg1", {}), ("cfg2", {"levels": 2}), ("cfg5", {"levels": 1})])
def test_square_transform_equals_subspace_sum(cfg, kw):
    """sum_alpha T_a (T_a^T R T_a / D_a) T_a^T == T (T^T R T / D) T^T  (SURVEY 8a a7 identity)."""
    pr, setup, f = get_setup(cfg, **kw)
    L = setup.finest
    smo = setup.smoother[L]
    scms = getattr(smo, "scms", smo)
    piece, solver = scms.interiors[0]
    rng = np.random.default_rng(3)
    R = rng.standard_normal(solver.dims)
    ref = np.zeros_like(R)
    for Ts, denom in solver._subspaces:
        Y = R
        for a, T in enumerate(Ts):
            Y = np.moveaxis(np.tensordot(T.T, Y, axes=(1, a)), 0, a)
        Y = Y / denom
        for a, T in enumerate(Ts):
            Y = np.moveaxis(np.tensordot(T, Y, axes=(1, a)), 0, a)
        ref += Y
    Ts, D = solver.square_transforms, solver.denominator
    Y = R
    for a, T in enumerate(Ts):
        Y = np.moveaxis(np.tensordot(T.T, Y, axes=(1, a)), 0, a)
    Y = Y / D
    for a, T in enumerate(Ts):
        Y = np.moveaxis(np.tensordot(T, Y, axes=(1, a)), 0, a)
    assert np.abs(Y - ref).max() <= 1e-13 * np.abs(ref).max()


def test_piece_inverse_matches_factorization():
    pr, setup, f = get_setup("cfg2", levels=2)
    scms = setup.smoother[2].scms
    A = setup.A[2].tocsr()
    for (piece, fact), inv in zip(scms.pieces, scms.piece_inverses):
        sub = A[piece.indices][:, piece.indices].toarray()
        assert np.abs(sub @ inv - np.eye(len(piece.indices))).max() <= 1e-10


def test_coarse_factor_convention():
    pr, setup, f = get_setup("cfg3", levels=2)
    L, U, pr_, pc = setup.coarse_solver.factors()
    b = np.random.default_rng(5).standard_normal(L.shape[0])
    import scipy.sparse.linalg as sla
    y = np.empty_like(b)
    y[pr_] = b
    w = sla.spsolve_triangular(U, sla.spsolve_triangular(L, y, lower=True), lower=False)
    x = w[pc]
    assert np.linalg.norm(setup.A[0] @ x - b) <= 1e-10 * np.linalg.norm(b)
    assert np.allclose(L.diagonal(), 1.0)


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference not present")
def test_matrices_equal_reference_directly():
    sys.path.insert(0, REFERENCE_SRC)
    from igamg import assembly as ra, geometry as rg, multigrid as rm
    dom = rg.l_shape()
    hier = ra.build_hierarchy(dom, 3, 2, "dg", coarse_elements=2)
    rs = rm.MultigridSolver(hier, rm.CycleConfig(smoother="hyb"))
    from paper_1902_01818_b200 import assembly as ma, geometry as mg, multigrid as mm
    h2 = ma.build_hierarchy(mg.l_shape(), 3, 2, "dg", coarse_elements=2)
    ms = mm.MultigridSetup(h2, mm.CycleConfig(smoother="hyb"))
    for l in range(3):
        d = abs(rs.A[l] - ms.A[l])
        assert (d.max() if d.nnz else 0.0) <= 1e-13 * abs(rs.A[l]).max()
    for l in range(1, 3):
        assert abs(rs.P[l] - ms.P[l]).nnz == 0


@pytest.mark.parametrize("name,kw", [("cfg1", {}), ("cfg2", {"levels": 3}), ("cfg3", {"levels": 2}),
                                     ("cfg4", {"p": 4, "levels": 2}), ("cfg5", {"levels": 1})])
def test_kronecker_transfer_description_reproduces_P(name, kw):
    """The per-patch Kronecker description the device transfer uses (1-D two-scale matrices,
    block maps, owner copies) reproduces the reference-form P and P^T to rounding."""
    from paper_1902_01818_b200 import assembly, configs
    pr = configs.build(name, **kw)
    rng = np.random.default_rng(4)
    for level in range(1, pr.hier.L + 1):
        P = assembly.prolongation(pr.hier, level)
        kd = assembly.prolongation_kron(pr.hier, level)
        assert kd["fine_owner"][kd["fine_free"] >= 0].sum() == P.shape[0]
        x, y = rng.standard_normal(P.shape[1]), rng.standard_normal(P.shape[0])
        assert np.abs(assembly.kron_apply(kd, x) - P @ x).max() <= 1e-14 * np.abs(P @ x).max()
        assert np.abs(assembly.kron_apply(kd, y, True) - P.T @ y).max() <= 1e-14 * np.abs(P.T @ y).max()


@pytest.mark.parametrize("name,kw", [("cfg5", {"levels": 2}), ("cfg2", {"levels": 3})])
def test_galerkin_equals_rediscretised_on_affine_patches(name, kw):
    """The matrix-free operator applies the rediscretised coarse operators; on nested spaces over
    affine patches they equal the reference's Galerkin products P^T A P (multigrid.py:95-99)."""
    from paper_1902_01818_b200 import assembly
    pr, setup, f = get_setup(name, **kw)
    for level in range(1, pr.hier.L):
        Ag, Ad = setup.A[level], assembly.assemble_level(pr.hier, level).A
        assert abs(Ag - Ad).max() <= 1e-14 * abs(Ag).max()


@pytest.mark.parametrize("cfg,kw", [("cfg1", {}), ("cfg2", {"levels": 2}), ("cfg5", {"levels": 1}),
                                    ("cfg5", {"levels": 2})])
def test_native_kron_assembly_bitwise(cfg, kw, monkeypatch):
    """csrc/host_setup.cpp's Kronecker assembly + free-DoF reduction equals the SciPy path array for
    array (indptr, indices, data), for A and the Dirichlet coupling (reference assembly.py:333-344,
    568-608)."""
    from paper_1902_01818_b200 import _setup_native, assembly, configs
    if _setup_native.lib() is None:
        pytest.skip("libigb_setup.so not built")
    pr = configs.build(cfg, **kw)
    for level in range(pr.hier.L + 1):
        nat = assembly.assemble_level(pr.hier, level)
        monkeypatch.setenv("IGB_NATIVE_SETUP", "0")
        ref = assembly.assemble_level(pr.hier, level)
        monkeypatch.delenv("IGB_NATIVE_SETUP")
        for a, b in ((nat.A, ref.A), (nat.couple, ref.couple)):
            a, b = a.tocsr(), b.tocsr()
            assert a.shape == b.shape
            assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices), (cfg, level)
            assert np.array_equal(a.data, b.data), (cfg, level, np.abs(a.data - b.data).max())


@pytest.mark.parametrize("cfg,kw", [("cfg2", {"levels": 3}), ("cfg3", {"levels": 2}), ("cfg4", {"p": 3, "levels": 2}),
                                    ("cfg5", {"levels": 2})])
def test_native_galerkin_bitwise(cfg, kw):
    """csrc/host_setup.cpp's P^T A P equals SciPy's (P.T @ A @ P).tocsr() bit for bit (multigrid.py:95-99)."""
    from paper_1902_01818_b200 import _setup_native, assembly, configs
    if _setup_native.lib() is None:
        pytest.skip("libigb_setup.so not built")
    pr = configs.build(cfg, **kw)
    A = assembly.assemble_level(pr.hier, pr.hier.L).A
    for level in range(pr.hier.L, 0, -1):
        P = assembly.prolongation(pr.hier, level)
        ref = (P.T @ A @ P).tocsr()
        ref.sort_indices()
        nat = _setup_native.galerkin(A, P)
        assert np.array_equal(nat.indptr, ref.indptr) and np.array_equal(nat.indices, ref.indices), (cfg, level)
        assert np.array_equal(nat.data, ref.data), (cfg, level, np.abs(nat.data - ref.data).max())
        A = ref
