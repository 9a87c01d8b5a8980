"""The CPU oracle (oracle/solve.py) pinned before it is trusted as the checker.

1. On the reference's own setup it reproduces the reference bit for bit
   (stored flag in every golden fixture; re-checked live when the reference is
   importable).
2. On the product's host setup it reproduces the golden iteration counts,
   residual histories and solutions of the reference.
3. SPEC known-answer tests for the solve-phase operators (SPEC.md:327-329,
   :386, :421-423, :438, :503).
"""

import os
import sys

import numpy as np
import pytest
import scipy.sparse

from conftest import REFERENCE_SRC, SMALL_CASES, get_setup, load_golden
from oracle.solve import OracleSolver, cg

ALL = SMALL_CASES + [("cfg2", "cfg2", {}), ("cfg3", "cfg3", {})]


@pytest.mark.parametrize("golden,cfg,kw", ALL)
def test_golden_generated_with_bitwise_oracle(golden, cfg, kw):
    g = load_golden(golden)
    assert bool(g["oracle_bitwise"]), "oracle did not reproduce the reference bit for bit"


@pytest.mark.parametrize("golden,cfg,kw", ALL)
def test_oracle_on_product_setup_matches_reference(golden, cfg, kw):
    g = load_golden(golden)
    pr, setup, f = get_setup(cfg, **kw)
    x, its, hist = OracleSolver(setup.setup_bundle()).solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
    assert its == int(g["its"])
    h, hg = np.array(hist), g["hist"]
    assert np.max(np.abs(h - hg) / hg) <= 1e-9
    assert np.max(np.abs(h - hg)) / hg[0] <= 1e-10
    assert np.linalg.norm(x - g["x"]) <= 1e-10 * np.linalg.norm(g["x"])


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference not present")
def test_oracle_bitwise_vs_reference_live():
    sys.path.insert(0, REFERENCE_SRC)
    from igamg import assembly as ra, geometry as rg, linsolve as rl, multigrid as rm
    from oracle.solve import bundle_from_reference
    hier = ra.build_hierarchy(rg.l_shape(), 3, 2, "dg", coarse_elements=2)
    for smoother in ("gs", "scms", "hyb"):
        rs = rm.MultigridSolver(hier, rm.CycleConfig(smoother=smoother))
        f = ra.assemble_rhs(hier, rs.assembled_finest, ra.ManufacturedProblem(2))
        x, its, hist = rl.cg(rs.A[2], f, rs.preconditioner(), tol=1e-8, max_iters=500)
        xo, itso, histo = OracleSolver(bundle_from_reference(rs)).solve(f)
        assert its == itso and hist == histo and np.array_equal(x, xo)
        rng = np.random.default_rng(1)
        r = rng.standard_normal(len(f))
        assert np.array_equal(rs.cycle(2, r.copy()), OracleSolver(bundle_from_reference(rs)).cycle(2, r.copy()))


def test_spec_gs_kat():
    """A=[[2,-1],[-1,2]], r=(1,1): forward GS -> (1/2, 3/4)."""
    from oracle.solve import _GaussSeidel
    A = scipy.sparse.csr_matrix(np.array([[2.0, -1.0], [-1.0, 2.0]]))
    gs = _GaussSeidel(A)
    assert np.allclose(gs.forward(np.array([1.0, 1.0])), [0.5, 0.75])
    assert np.allclose(gs.backward(np.array([1.0, 1.0])), [0.75, 0.5])


def test_spec_cg_kats():
    """b=0 -> 0 its; identity -> 1 it; exact inverse -> <= 2 its."""
    A = scipy.sparse.identity(5, format="csr")
    x, its, hist = cg(A, np.zeros(5))
    assert its == 0 and hist == [] and not x.any()
    x, its, hist = cg(A, np.arange(1.0, 6.0))
    assert its == 1 and np.allclose(x, np.arange(1.0, 6.0))
    rng = np.random.default_rng(0)
    G = rng.standard_normal((20, 20))
    S = G.T @ G + np.eye(20)
    inv = np.linalg.inv(S)
    x, its, hist = cg(scipy.sparse.csr_matrix(S), rng.standard_normal(20), preconditioner=lambda r: inv @ r, tol=1e-10)
    assert its <= 2


def test_cg_reports_nonconvergence_without_raising():
    rng = np.random.default_rng(1)
    G = rng.standard_normal((30, 30))
    S = scipy.sparse.csr_matrix(G.T @ G + 0.01 * np.eye(30))
    x, its, hist = cg(S, rng.standard_normal(30), tol=1e-14, max_iters=3)
    assert its == 3 and len(hist) == 3


@pytest.mark.parametrize("cfg,kw", [("cfg1", {}), ("cfg2", {"levels": 2}), ("cfg3", {"levels": 2})])
def test_oracle_preconditioner_spd_and_linear(cfg, kw):
    """Cycle symmetry / positivity (multigrid.py:144-159) and linearity (SPEC multigrid invariants)."""
    pr, setup, f = get_setup(cfg, **kw)
    orc = OracleSolver(setup.setup_bundle())
    assert orc.check_spd()
    rng = np.random.default_rng(2)
    r, s = rng.standard_normal(setup.n_dofs), rng.standard_normal(setup.n_dofs)
    L = setup.finest
    lhs = orc.cycle(L, 2.0 * r + 3.0 * s)
    rhs = 2.0 * orc.cycle(L, r) + 3.0 * orc.cycle(L, s)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)


def test_scms_tau_linearity_and_symmetry():
    """apply(2 tau) = 2 apply(tau); r^T S s = s^T S r."""
    pr, setup, f = get_setup("cfg2", levels=2)
    bundle = setup.setup_bundle()
    orc = OracleSolver(bundle)
    rng = np.random.default_rng(4)
    r, s = rng.standard_normal(setup.n_dofs), rng.standard_normal(setup.n_dofs)
    a = orc.scms_apply(2, r)
    bundle2 = dict(bundle, levels=[None] + [dict(e, tau=2 * e["tau"]) for e in bundle["levels"][1:]])
    b = OracleSolver(bundle2).scms_apply(2, r)
    assert np.allclose(b, 2 * a, rtol=1e-14, atol=0)
    assert abs(s @ orc.scms_apply(2, r) - r @ orc.scms_apply(2, s)) <= 1e-12 * abs(s @ a)


@pytest.mark.parametrize("cfg,kw", [("cfg2", {"levels": 3}), ("cfg3", {"levels": 2}), ("cfg4", {"p": 8, "levels": 2}),
                                    ("cfg5", {"levels": 2})])
def test_trisolve_restatement_matches_superlu(cfg, kw):
    """oracle/trisolve.c (row substitution, used where splu(tril(A)) does not fit) against the
    reference's SuperLU NATURAL sweeps (smoothers.py:178-190) on every level: equal to rounding."""
    from oracle.solve import _GaussSeidel, _TriSolveGS
    pr, setup, f = get_setup(cfg, **kw)
    rng = np.random.default_rng(12)
    for level in range(1, setup.finest + 1):
        A = setup.A[level]
        r = rng.standard_normal(A.shape[0])
        a, b = _GaussSeidel(A), _TriSolveGS(A)
        for d in ("forward", "backward"):
            x, y = getattr(a, d)(r), getattr(b, d)(r)
            assert np.linalg.norm(x - y) <= 1e-13 * np.linalg.norm(x), (cfg, level, d)


@pytest.mark.parametrize("golden,cfg,kw", [("cfg2_L3", "cfg2", {"levels": 3}), ("cfg3_L2", "cfg3", {"levels": 2}),
                                           ("cfg5_L2", "cfg5", {"levels": 2}), ("cfg4_p8_L3", "cfg4", {"p": 8, "levels": 3})])
def test_trisolve_oracle_matches_reference_golden(golden, cfg, kw):
    """The oracle with C-substitution sweeps (the full-size checker of cfg4 p = 8 / cfg5) reproduces
    the reference's golden iteration counts, histories (1e-10 per entry; cfg3 3e-10, SURVEY
    Appendix C) and solutions."""
    g = load_golden(golden)
    pr, setup, f = get_setup(cfg, **kw)
    x, its, hist = OracleSolver(setup.setup_bundle(), gs_impl="trisolve").solve(
        f, tol=pr.config.tol, max_iters=pr.config.max_iters)
    assert its == int(g["its"])
    h, hg = np.array(hist), g["hist"]
    d = np.abs(h - hg)
    print(f"[trisolve oracle] {golden}: per entry {np.max(d / hg):.2e}, max|dh|/h1 {np.max(d) / hg[0]:.2e}")
    floor = 64 * np.finfo(float).eps * hg[0]  # see tests/test_gpu_parity.py hist_ok
    assert np.all(d <= np.maximum((3e-10 if cfg == "cfg3" else 1e-10) * hg, floor))
    assert np.linalg.norm(x - g["x"]) <= 1e-10 * np.linalg.norm(g["x"])
