"""The rest of the drop-in surface and the secondary drivers, on the device vs the oracle.

* ``linsolve.cg`` with ``preconditioner=None``, with a host callable, and with the device
  preconditioner plus a live per-iteration ``callback`` (reference linsolve.py:64-101);
* the smoother duck type ``pre_smooth`` / ``post_smooth(A, u, f, steps)`` of GaussSeidel,
  SubspaceCorrectedMass and HybridSmoother (smoothers.py:192-200, 327-332, 343-353);
* ``MultigridSolver.cycle(level, f, u)`` from a nonzero iterate (multigrid.py:118-138);
* ``solve_stationary`` / ``solve_direct`` iterates (multigrid.py:202-234), the 'theory' smoothing
  schedule (multigrid.py:46-50), and the triangular coarse path (``IGB_COARSE=csc``, the method
  north-star item (5) names) against the oracle.
"""

import dataclasses
import os

import numpy as np
import pytest

from conftest import get_setup
from test_gpu_parity import hist_ok

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


_cache = {}


def solver_for(cfg, **kw):
    key = (cfg, tuple(sorted(kw.items())))
    if key not in _cache:
        from paper_1902_01818_b200 import multigrid
        from oracle.solve import OracleSolver
        pr, setup, f = get_setup(cfg, **kw)
        _cache[key] = (pr, setup, f, multigrid.MultigridSolver(pr.hier, pr.config, device=0, setup=setup),
                       OracleSolver(setup.setup_bundle()))
    return _cache[key]


def test_cg_plain_host_callable_and_live_callback():
    from oracle.solve import cg as ocg
    from paper_1902_01818_b200 import linsolve
    pr, setup, f, solver, orc = solver_for("cfg1", levels=1)
    A = solver.A[solver.finest]
    # plain CG (a random right-hand side: the configuration's own f is an eigenvector of the
    # single-patch operator, so plain CG on it stops after one step at rounding-noise level)
    fr = np.random.default_rng(1).standard_normal(len(f))
    x, its, h = linsolve.cg(A, fr, None, tol=1e-8, max_iters=2000)
    xo, itso, ho = ocg(A, fr, None, tol=1e-8, max_iters=2000)
    assert its == itso
    assert np.max(np.abs(np.array(h) - ho)) / ho[0] <= 1e-10
    assert rel(x, xo) <= 1e-8
    # host callable preconditioner (Jacobi)
    dinv = 1.0 / A.diagonal()
    jac = lambda r: dinv * r  # noqa: E731
    x, its, h = linsolve.cg(A, fr, jac, tol=1e-8, max_iters=2000)
    xo, itso, ho = ocg(A, fr, jac, tol=1e-8, max_iters=2000)
    assert its == itso
    assert np.max(np.abs(np.array(h) - ho)) / ho[0] <= 1e-10
    assert rel(x, xo) <= 1e-8
    # device preconditioner with a live callback: called once per iteration, during the solve
    seen = []
    x, its, h = linsolve.cg(A, f, solver.preconditioner(), tol=1e-8, max_iters=500,
                            callback=lambda it, r: seen.append((it, r)))
    assert [s[0] for s in seen] == list(range(1, its + 1))
    assert [s[1] for s in seen] == h
    xo, itso, ho = orc.solve(f)
    # the last entry of this one-level solve is 2e-16 (rounding noise): floor-aware comparison
    assert its == itso and hist_ok(h, ho)[0], hist_ok(h, ho)


def test_smoother_duck_type_matches_oracle():
    pr, setup, f, solver, orc = solver_for("cfg3", levels=2)
    L = solver.finest
    A = solver.A[L]
    smo = solver.smoother[L]
    rng = np.random.default_rng(19)
    u0, rhs = rng.standard_normal(A.shape[0]), rng.standard_normal(A.shape[0])
    # GaussSeidel: steps of u += GS_fwd(f - A u) / GS_bwd
    for post, ref in ((False, orc.gs_forward), (True, orc.gs_backward)):
        u = u0.copy()
        want = u0.copy()
        for _ in range(2):
            want = want + ref(L, rhs - A @ want)
        out = smo.gs.post_smooth(A, u, rhs, 2) if post else smo.gs.pre_smooth(A, u, rhs, 2)
        assert out is u and rel(u, want) <= 1e-12
    # SubspaceCorrectedMass
    u = u0.copy()
    want = u0.copy()
    for _ in range(2):
        want = want + orc.scms_apply(L, rhs - A @ want)
    smo.scms.pre_smooth(A, u, rhs, 2)
    assert rel(u, want) <= 1e-12
    # HybridSmoother (pre: GS then SCMS; post: SCMS then GS)
    for post in (False, True):
        u = u0.copy()
        want = (orc._post if post else orc._pre)(L, A, u0.copy(), rhs, 1)
        (smo.post_smooth if post else smo.pre_smooth)(A, u, rhs, 1)
        assert rel(u, want) <= 1e-12


def test_cycle_from_nonzero_iterate():
    pr, setup, f, solver, orc = solver_for("cfg2", levels=3)
    L = solver.finest
    u = np.random.default_rng(23).standard_normal(solver.n_dofs)
    assert rel(solver.cycle(L, f, u.copy()), orc.cycle(L, f, u.copy())) <= 1e-11


@pytest.mark.parametrize("mode", ["stationary", "direct"])
def test_stationary_and_direct_iterates_match_oracle(mode):
    pr, setup, f, solver, orc = solver_for("cfg2", levels=3)
    rep = solver.solve(f, mode=mode)
    uo, itso, reso, conv = getattr(orc, f"solve_{mode}")(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
    assert rep.iterations == itso and rep.converged == conv
    h, ho = np.array(rep.residuals), np.array(reso)
    assert np.max(np.abs(h - ho)) / ho[0] <= 1e-10
    # residuals of the stationary iteration are f - A u recomputed from u: their absolute rounding
    # noise is ~1e-13 of the first one, whatever their size
    assert np.all(np.abs(h - ho) <= np.maximum(1e-8 * ho, 1e-13 * ho[0]))
    assert rel(rep.x, uo) <= 1e-9


def test_theory_schedule_matches_oracle():
    from paper_1902_01818_b200 import multigrid
    from oracle.solve import OracleSolver
    pr, _, _ = get_setup("cfg2", levels=2)
    cfg = dataclasses.replace(pr.config, nu_schedule="theory")
    setup = multigrid.MultigridSetup(pr.hier, cfg)
    assert setup.setup_bundle()["steps"][1] > 1  # the coarser level smooths more
    f = pr.rhs(setup.assembled_finest)
    solver = multigrid.MultigridSolver(pr.hier, cfg, device=0, setup=setup)
    orc = OracleSolver(setup.setup_bundle())
    rep = solver.solve_pcg(f)
    xo, itso, histo = orc.solve(f, tol=cfg.tol, max_iters=cfg.max_iters)
    assert rep.iterations == itso
    assert np.max(np.abs(np.array(rep.residuals) - histo) / np.array(histo)) <= 1e-10
    assert rel(rep.x, xo) <= 1e-10
    solver.close()


def test_triangular_coarse_path_matches_oracle():
    from paper_1902_01818_b200 import multigrid
    from oracle.solve import OracleSolver
    pr, setup, f = get_setup("cfg3", levels=2)
    os.environ["IGB_COARSE"] = "csc"
    try:
        solver = multigrid.MultigridSolver(pr.hier, pr.config, device=0, setup=setup)
    finally:
        del os.environ["IGB_COARSE"]
    orc = OracleSolver(setup.setup_bundle())
    x0 = np.random.default_rng(29).standard_normal(solver.A[0].shape[0])
    assert rel(solver.ctx.op("coarse", 0, x0, len(x0)), orc.coarse_solve(x0)) <= 1e-11
    rep = solver.solve_pcg(f)
    xo, itso, histo = orc.solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
    assert rep.iterations == itso
    assert np.max(np.abs(np.array(rep.residuals) - histo) / np.array(histo)) <= 3e-10  # SIPG floor
    assert rel(rep.x, xo) <= 1e-10
    solver.close()
