"""Device parity: every hot-path operator and the whole PCG solve vs the oracle.

Calls go through the C-ABI (libigb.so via ctypes).  Tolerances:
  * single operators (A@x, P@e, P^T r, GS sweeps, SCMS apply, coarse solve,
    one cycle): relative 2-norm difference <= 1e-12 (fp64, summation-order noise);
  * PCG: identical iteration counts; residual history per entry |dh_i| / h_i <= 1e-10
    (the north star's bound; an entry whose |dh_i| is within 64 ulps of h_1 -- the rounding floor
    of a relative residual -- passes: see hist_ok) and max_i |dh_i| / h_1 <= 1e-10; solution
    ||dx|| / ||x|| <= 1e-10.
    Exception: the SIPG L-shape (cfg3 family) is held to 3e-10 per entry -- SURVEY Appendix C
    measured 3.5e-10 there for a CPU restatement that only re-orders sums (cond(A_0) = 1.2e6,
    the over-penalised coarse SIPG operator); this build measures 2.1e-10 (profiles/r1l_configs.jsonl);
  * against the reference's own golden histories the same bounds apply.
"""

import numpy as np
import pytest

from conftest import SMALL_CASES, get_setup, load_golden

pytestmark = pytest.mark.gpu

_solvers = {}


def device_solver(cfg, **kw):
    key = (cfg, tuple(sorted(kw.items())))
    if key not in _solvers:
        from paper_1902_01818_b200 import multigrid
        from oracle.solve import OracleSolver
        pr, setup, f = get_setup(cfg, **kw)
        solver = multigrid.MultigridSolver(pr.hier, pr.config, device=0, setup=setup)
        _solvers[key] = (pr, setup, f, solver, OracleSolver(setup.setup_bundle()))
    return _solvers[key]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


OP_CASES = [(c, k) for _, c, k in SMALL_CASES] + [("cfg2", {})]


@pytest.mark.parametrize("cfg,kw", OP_CASES)
def test_operators_match_oracle(cfg, kw):
    pr, setup, f, solver, orc = device_solver(cfg, **kw)
    ctx = solver.ctx
    rng = np.random.default_rng(11)
    for level in range(1, solver.finest + 1):
        n = solver.A[level].shape[0]
        nc = solver.A[level - 1].shape[0]
        x = rng.standard_normal(n)
        assert rel(ctx.op("spmv", level, x, n), solver.A[level] @ x) <= 1e-12
        fres = rng.standard_normal(n)
        assert rel(ctx.op("residual", level, x, n, out_init=fres), fres - solver.A[level] @ x) <= 1e-12
        if orc.gs[level] is not None:
            assert rel(ctx.op("gs_fwd", level, x, n), orc.gs_forward(level, x)) <= 1e-12
            assert rel(ctx.op("gs_bwd", level, x, n), orc.gs_backward(level, x)) <= 1e-12
        if orc.scms[level] is not None:
            assert rel(ctx.op("scms", level, x, n), orc.scms_apply(level, x)) <= 1e-12
        assert rel(ctx.op("restrict", level, x, nc), solver.P[level].T @ x) <= 1e-12
        xc = rng.standard_normal(nc)
        assert rel(ctx.op("prolong", level, xc, n), solver.P[level] @ xc) <= 1e-12
        assert rel(ctx.op("cycle", level, x, n), orc.cycle(level, x)) <= 1e-11
    x0 = rng.standard_normal(solver.A[0].shape[0])
    assert rel(ctx.op("coarse", 0, x0, len(x0)), orc.coarse_solve(x0)) <= 1e-11


HIST_TOL = 1e-10
HIST_TOL_SIPG = 3e-10  # cfg3 family: the fp64 floor of SURVEY Appendix C (see module docstring)
# A history entry is ||r_i|| / ||b||; its absolute rounding noise is a few ulps of the initial
# relative residual h_1 whatever its size, so an entry far below h_1 (cfg4 p = 8: 4e-9 after 11
# iterations) cannot be compared to 1e-10 of itself.  Entries whose absolute difference is within
# 64 ulps of h_1 (1.4e-14 h_1, 7000x tighter than round 1's h_1-relative 1e-10 bound) pass.
HIST_FLOOR_ULPS = 64


def hist_tol(cfg):
    return HIST_TOL_SIPG if cfg == "cfg3" else HIST_TOL


def hist_ok(h, ho, per_entry=HIST_TOL):
    """(ok, max per-entry relative difference, max |dh| / h_1) with the floor above."""
    h, ho = np.asarray(h), np.asarray(ho)
    d = np.abs(h - ho)
    bound = np.maximum(per_entry * ho, HIST_FLOOR_ULPS * np.finfo(float).eps * ho[0])
    return bool(np.all(d <= bound)), float(np.max(d / ho)), float(np.max(d) / ho[0])


def _check_history(h, ho, tag, per_entry=HIST_TOL):
    h, ho = np.asarray(h), np.asarray(ho)
    assert len(h) == len(ho), tag
    ok, de, d1 = hist_ok(h, ho, per_entry)
    print(f"[hist] {tag}: max|dh|/h1 {d1:.2e}  per entry {de:.2e}")
    assert d1 <= 1e-10, (tag, d1)
    assert ok, (tag, de, d1)


@pytest.mark.parametrize("golden,cfg,kw", SMALL_CASES + [("cfg2", "cfg2", {}), ("cfg3", "cfg3", {})])
def test_pcg_matches_oracle_and_reference(golden, cfg, kw):
    pr, setup, f, solver, orc = device_solver(cfg, **kw)
    rep = solver.solve_pcg(f)
    xo, itso, histo = orc.solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
    assert rep.iterations == itso and rep.converged
    _check_history(rep.residuals, histo, f"{golden} vs oracle", hist_tol(cfg))
    assert rel(rep.x, xo) <= 1e-10
    g = load_golden(golden)
    assert rep.iterations == int(g["its"])
    _check_history(rep.residuals, g["hist"], f"{golden} vs reference golden", hist_tol(cfg))
    assert rel(rep.x, g["x"]) <= 1e-10


def test_linsolve_cg_dropin_and_determinism():
    from paper_1902_01818_b200 import linsolve
    pr, setup, f, solver, orc = device_solver("cfg2", levels=3)
    L = solver.finest
    calls = []
    x1, its1, h1 = linsolve.cg(solver.A[L], f, solver.preconditioner(), tol=1e-8, max_iters=500,
                               callback=lambda it, rel_: calls.append(it))
    x2, its2, h2 = linsolve.cg(solver.A[L], f, solver.preconditioner(), tol=1e-8, max_iters=500)
    assert its1 == its2 and h1 == h2 and np.array_equal(x1, x2), "device solve is not bitwise reproducible"
    assert calls == list(range(1, its1 + 1))
    xr, itsr, hr = linsolve.cg(solver.A[L], f, solver.preconditioner(), tol=1e-14, max_iters=3)
    assert itsr == 3 and len(hr) == 3


def test_zero_rhs_and_spd_check():
    pr, setup, f, solver, orc = device_solver("cfg1")
    rep = solver.solve_pcg(np.zeros_like(f))
    assert rep.iterations == 0 and rep.residuals == [] and not rep.x.any()
    solver.check_preconditioner_spd()


def test_cycle_linearity_and_symmetry_on_device():
    pr, setup, f, solver, orc = device_solver("cfg3", levels=2)
    L = solver.finest
    rng = np.random.default_rng(5)
    r, s = rng.standard_normal(solver.n_dofs), rng.standard_normal(solver.n_dofs)
    Br, Bs = solver.cycle(L, r), solver.cycle(L, s)
    assert abs(s @ Br - r @ Bs) <= 1e-10 * abs(s @ Br)
    assert rel(solver.cycle(L, 2.0 * r + 3.0 * s), 2.0 * Br + 3.0 * Bs) <= 1e-12


def test_stationary_and_direct_drivers():
    pr, setup, f, solver, orc = device_solver("cfg2", levels=3)
    for mode in ("stationary", "direct"):
        rep = solver.solve(f, mode=mode)
        assert rep.converged and rep.residuals[-1] <= 1e-8
        assert np.linalg.norm(solver.A[solver.finest] @ rep.x - f) <= 1e-7 * np.linalg.norm(f)


def test_smoother_objects_apply_on_device():
    pr, setup, f, solver, orc = device_solver("cfg2", levels=2)
    smo = solver.smoother[2]
    rng = np.random.default_rng(6)
    r = rng.standard_normal(solver.A[2].shape[0])
    assert rel(smo.gs.apply_forward(r), orc.gs_forward(2, r)) <= 1e-12
    assert rel(smo.scms.apply(r), orc.scms_apply(2, r)) <= 1e-12


def test_bad_arguments_are_errors():
    from paper_1902_01818_b200._lib import Context, IgbError
    ctx = Context(0)
    with pytest.raises(IgbError):
        ctx.set_num_levels(0)
    ctx.set_num_levels(1)
    import scipy.sparse
    bad = scipy.sparse.csr_matrix(np.array([[1.0, 2.0], [0.0, 0.0]]))
    with pytest.raises(IgbError):
        ctx.set_level_matrix(1, bad)   # zero diagonal
    with pytest.raises(IgbError):
        ctx.finalize()                 # incomplete hierarchy
    ctx.close()


@pytest.mark.slow
@pytest.mark.parametrize("golden,cfg,kw", [("cfg4_p2", "cfg4", {"p": 2}), ("cfg4_p4", "cfg4", {"p": 4}),
                                            ("cfg5_L3", "cfg5", {"levels": 3})])
def test_large_configs_match_reference_golden(golden, cfg, kw):
    """Large configurations against the reference run here (tools/make_golden.py): cfg4 at full size
    (p = 2: N = 1,054,729, 26M nnz; p = 4: N = 1,071,225, 86M nnz; 16 distorted patches, 7 levels) and
    cfg5 at L = 3 (3-D, N = 300,763, 92M nnz; flow sweeps on every level).  Iteration count, the
    residual history and a strided sample of x (and of f, pinning the host setup)."""
    g = load_golden(golden)
    from paper_1902_01818_b200 import multigrid
    pr, setup, f = get_setup(cfg, **kw)
    step = int(g["x_sample_step"])
    assert np.abs(f[::step] - g["f_sample"]).max() <= 1e-13 * np.abs(g["f_sample"]).max()
    solver = multigrid.MultigridSolver(pr.hier, pr.config, device=0, setup=setup)
    rep = solver.solve_pcg(f, check_spd=False)
    assert rep.iterations == int(g["its"])
    _check_history(rep.residuals, g["hist"], f"{golden} vs reference golden")
    xs = rep.x[::step]
    assert np.linalg.norm(xs - g["x_sample"]) <= 1e-10 * np.linalg.norm(g["x_sample"])
    solver.close()


def test_gs_cluster_path_matches_oracle():
    """Force the clustered sweep on a small level (IGB_GS_CLUSTER) and compare with SuperLU."""
    import os
    from paper_1902_01818_b200 import multigrid
    from oracle.solve import OracleSolver
    pr, setup, f = get_setup("cfg3", levels=2)
    os.environ["IGB_GS_FORCE_CLUSTER"] = "3"
    try:
        solver = multigrid.MultigridSolver(pr.hier, pr.config, device=0, setup=setup)
    finally:
        del os.environ["IGB_GS_FORCE_CLUSTER"]
    orc = OracleSolver(setup.setup_bundle())
    rng = np.random.default_rng(9)
    for level in (1, 2):
        n = solver.A[level].shape[0]
        x = rng.standard_normal(n)
        assert rel(solver.ctx.op("gs_fwd", level, x, n), orc.gs_forward(level, x)) <= 1e-12
        assert rel(solver.ctx.op("gs_bwd", level, x, n), orc.gs_backward(level, x)) <= 1e-12
    solver.close()


STRESS_CASES = [("cfg2", {}), ("cfg3", {"levels": 3}), ("cfg4", {"p": 4, "levels": 3}), ("cfg5", {"levels": 2})]


@pytest.mark.parametrize("cfg,kw", STRESS_CASES)
def test_gs_sweeps_repeatable_and_match_oracle(cfg, kw):
    """Every level's forward/backward sweep, 12 repetitions each: bitwise identical results
    (the panel sweep's cluster exchanges are race-free and its reductions fixed-order) and
    within 1e-12 of SuperLU on tril/triu."""
    pr, setup, f, solver, orc = device_solver(cfg, **kw)
    rng = np.random.default_rng(17)
    for level in range(1, solver.finest + 1):
        if orc.gs[level] is None:
            continue
        n = solver.A[level].shape[0]
        x = rng.standard_normal(n)
        for op, ref in (("gs_fwd", orc.gs_forward), ("gs_bwd", orc.gs_backward)):
            first = solver.ctx.op(op, level, x, n)
            for _ in range(11):
                assert np.array_equal(solver.ctx.op(op, level, x, n), first), (cfg, level, op)
            assert rel(first, ref(level, x)) <= 1e-12, (cfg, level, op)


def test_level_set_engine_still_matches_oracle():
    """IGB_GS_ENGINE=levels: the level-set sweep (used when panels do not pay off)."""
    import os
    from paper_1902_01818_b200 import multigrid
    from oracle.solve import OracleSolver
    pr, setup, f = get_setup("cfg2", levels=3)
    os.environ["IGB_GS_ENGINE"] = "levels"
    try:
        solver = multigrid.MultigridSolver(pr.hier, pr.config, device=0, setup=setup)
    finally:
        del os.environ["IGB_GS_ENGINE"]
    orc = OracleSolver(setup.setup_bundle())
    rng = np.random.default_rng(3)
    for level in (1, 2, 3):
        n = solver.A[level].shape[0]
        x = rng.standard_normal(n)
        assert rel(solver.ctx.op("gs_fwd", level, x, n), orc.gs_forward(level, x)) <= 1e-12
        assert rel(solver.ctx.op("gs_bwd", level, x, n), orc.gs_backward(level, x)) <= 1e-12
    rep = solver.solve_pcg(f)
    xo, itso, histo = orc.solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
    assert rep.iterations == itso
    solver.close()


FLOW_CASES = [("cfg2", {"levels": 3}, None), ("cfg3", {"levels": 2}, None), ("cfg5", {"levels": 2}, None),
              ("cfg4", {"p": 4, "levels": 2}, "8"), ("cfg2", {"levels": 2}, "16")]


@pytest.mark.parametrize("cfg,kw,G", FLOW_CASES)
def test_flow_engine_matches_oracle(cfg, kw, G):
    """IGB_GS_ENGINE=flow: the dependency-driven whole-GPU sweep on every level (chosen
    automatically for wide levels: 3-D, high degree).  Each sweep 6x bitwise repeatable
    (fixed per-row summation order, parity-alternating sentinel copy), within 1e-12 of
    SuperLU on tril/triu, and the PCG solve matches the oracle."""
    import os
    from paper_1902_01818_b200 import multigrid
    from oracle.solve import OracleSolver
    pr, setup, f = get_setup(cfg, **kw)
    os.environ["IGB_GS_ENGINE"] = "flow"
    if G:
        os.environ["IGB_FLOW_G"] = G
    try:
        solver = multigrid.MultigridSolver(pr.hier, pr.config, device=0, setup=setup)
    finally:
        del os.environ["IGB_GS_ENGINE"]
        os.environ.pop("IGB_FLOW_G", None)
    orc = OracleSolver(setup.setup_bundle())
    rng = np.random.default_rng(23)
    for level in range(1, solver.finest + 1):
        if orc.gs[level] is None:
            continue
        n = solver.A[level].shape[0]
        x = rng.standard_normal(n)
        for op, ref in (("gs_fwd", orc.gs_forward), ("gs_bwd", orc.gs_backward)):
            first = solver.ctx.op(op, level, x, n)
            for _ in range(5):
                assert np.array_equal(solver.ctx.op(op, level, x, n), first), (cfg, level, op)
            assert rel(first, ref(level, x)) <= 1e-12, (cfg, level, op)
    rep = solver.solve_pcg(f)
    xo, itso, histo = orc.solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
    assert rep.iterations == itso
    _check_history(rep.residuals, histo, f"{cfg} flow vs oracle", hist_tol(cfg))
    assert rel(rep.x, xo) <= 1e-10
    solver.close()


@pytest.mark.parametrize("cfg,kw,ctas", [("cfg5", {"levels": 2}, None), ("cfg5", {"levels": 2}, "64"),
                                         ("cfg2", {"levels": 2}, None)])
def test_wave_engine_matches_oracle(cfg, kw, ctas):
    """IGB_GS_ENGINE=wave (opt-in): plane chains inside one CTA, external sums by the rest of the GPU
    (wave.cu, wave_plan.cpp).  Every sweep 6x bitwise repeatable and within 1e-12 of SuperLU on
    tril / triu, the PCG solve matches the oracle; with 64 CTAs the groups sweep several bundles
    each (ticket hand-out, queue reuse)."""
    import os
    from paper_1902_01818_b200 import multigrid
    from oracle.solve import OracleSolver
    pr, setup, f = get_setup(cfg, **kw)
    os.environ["IGB_GS_ENGINE"] = "wave"
    if ctas:
        os.environ["IGB_WAVE_CTAS"] = ctas
    try:
        solver = multigrid.MultigridSolver(pr.hier, pr.config, device=0, setup=setup)
    finally:
        del os.environ["IGB_GS_ENGINE"]
        os.environ.pop("IGB_WAVE_CTAS", None)
    orc = OracleSolver(setup.setup_bundle())
    rng = np.random.default_rng(29)
    engines = set()
    for level in range(1, solver.finest + 1):
        if orc.gs[level] is None:
            continue
        n = solver.A[level].shape[0]
        x = rng.standard_normal(n)
        for d, (op, ref) in enumerate((("gs_fwd", orc.gs_forward), ("gs_bwd", orc.gs_backward))):
            engines.add(solver.ctx.gs_info(level, d)["engine"])
            first = solver.ctx.op(op, level, x, n)
            for _ in range(5):
                assert np.array_equal(solver.ctx.op(op, level, x, n), first), (cfg, level, op)
            assert rel(first, ref(level, x)) <= 1e-12, (cfg, level, op)
    assert "wave" in engines
    rep = solver.solve_pcg(f)
    xo, itso, histo = orc.solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
    assert rep.iterations == itso
    _check_history(rep.residuals, histo, f"{cfg} wave vs oracle", hist_tol(cfg))
    assert rel(rep.x, xo) <= 1e-10
    solver.close()


@pytest.mark.parametrize("cfg,kw", [("cfg2", {"levels": 3}), ("cfg3", {"levels": 2}), ("cfg5", {"levels": 2}),
                                    ("cfg4", {"p": 4, "levels": 2})])
def test_kronecker_transfers_match_P(cfg, kw):
    """IGB_TRANSFER=kron: restriction / prolongation as per-patch Kronecker products of the 1-D
    two-scale matrices (transfer.cu) against the reference-form P, and the PCG solve on them."""
    import os
    from paper_1902_01818_b200 import multigrid
    from oracle.solve import OracleSolver
    pr, setup, f = get_setup(cfg, **kw)
    os.environ["IGB_TRANSFER"] = "kron"
    try:
        solver = multigrid.MultigridSolver(pr.hier, pr.config, device=0, setup=setup)
    finally:
        del os.environ["IGB_TRANSFER"]
    rng = np.random.default_rng(31)
    for level in range(1, solver.finest + 1):
        n, nc = solver.A[level].shape[0], solver.A[level - 1].shape[0]
        x, xc = rng.standard_normal(n), rng.standard_normal(nc)
        r1 = solver.ctx.op("restrict", level, x, nc)
        assert rel(r1, solver.P[level].T @ x) <= 1e-13
        assert np.array_equal(solver.ctx.op("restrict", level, x, nc), r1)  # fixed summation order
        assert rel(solver.ctx.op("prolong", level, xc, n), solver.P[level] @ xc) <= 1e-13
    orc = OracleSolver(setup.setup_bundle())
    rep = solver.solve_pcg(f)
    xo, itso, histo = orc.solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
    assert rep.iterations == itso
    _check_history(rep.residuals, histo, f"{cfg} kron transfers vs oracle", hist_tol(cfg))
    assert rel(rep.x, xo) <= 1e-10
    solver.close()


@pytest.mark.parametrize("smoother,nu,mu", [("gs", 2, 1), ("gs", 1, 2), ("hyb", 2, 1), ("scms", 1, 1)])
def test_other_smoothers_and_cycles_match_oracle(smoother, nu, mu):
    """Non-default cycle knobs (multigrid.py:23-50): plain Gauss-Seidel smoothing with nu = 2
    (forward steps from a nonzero iterate use T u' = f - (A - T) u), the W-cycle, the hybrid
    smoother with nu = 2, SCMS alone -- device PCG against the oracle on the same setup."""
    import dataclasses
    from paper_1902_01818_b200 import multigrid
    from oracle.solve import OracleSolver
    pr, _, _ = get_setup("cfg3", levels=2)
    cfg = dataclasses.replace(pr.config, smoother=smoother, nu=nu, mu=mu)
    setup = multigrid.MultigridSetup(pr.hier, cfg)
    f = pr.rhs(setup.assembled_finest)
    solver = multigrid.MultigridSolver(pr.hier, cfg, device=0, setup=setup)
    orc = OracleSolver(setup.setup_bundle())
    rng = np.random.default_rng(41)
    r = rng.standard_normal(solver.n_dofs)
    assert rel(solver.cycle(solver.finest, r), orc.cycle(solver.finest, r)) <= 1e-11
    rep = solver.solve_pcg(f)
    xo, itso, histo = orc.solve(f, tol=cfg.tol, max_iters=cfg.max_iters)
    assert rep.iterations == itso
    # not a BASELINE configuration: plain GS on the SIPG L-shape needs up to 28 iterations, and the
    # per-entry drift of the late (h ~ 1e-8) entries grows with the iteration count (measured 1.1e-9 for
    # the W-cycle, 2.7e-10 for nu = 2); the h_1-relative bound stays 1e-10
    _check_history(rep.residuals, histo, f"cfg3 {smoother} nu={nu} mu={mu}", 2e-9)
    assert rel(rep.x, xo) <= 1e-10
    solver.close()


def test_pinned_host_buffers_pcg_bitwise():
    """igb_pcg with page-locked host buffers (igb_host_alloc): same result, bit for bit, as with
    pageable numpy buffers and as the device-buffer entry point."""
    pr, setup, f, solver, orc = device_solver("cfg2", levels=3)
    ctx = solver.ctx
    x1, its1, h1 = ctx.pcg(f, 1e-8, 500)
    b, xo = ctx.pinned(len(f)), ctx.pinned(len(f))
    b[:] = f
    x2, its2, h2 = ctx.pcg(b, 1e-8, 500, out=xo)
    assert x2 is xo and its1 == its2 and h1 == h2 and np.array_equal(x1, x2)


def test_p8_backward_panel_matches_oracle():
    """cfg4 p = 8 (L = 3): backward rows carry ~200 near entries -- the panel variant with 14
    slots per lane (one range) -- sweeps repeatable and equal to SuperLU on triu(A) per level."""
    pr, setup, f, solver, orc = device_solver("cfg4", p=8, levels=3)
    rng = np.random.default_rng(43)
    for level in range(1, solver.finest + 1):
        n = solver.A[level].shape[0]
        x = rng.standard_normal(n)
        for op, ref in (("gs_fwd", orc.gs_forward), ("gs_bwd", orc.gs_backward)):
            first = solver.ctx.op(op, level, x, n)
            for _ in range(3):
                assert np.array_equal(solver.ctx.op(op, level, x, n), first), (level, op)
            assert rel(first, ref(level, x)) <= 1e-12, (level, op)


def test_standalone_gauss_seidel_helpers():
    """smoothers.gs_apply_forward / gs_apply_backward (reference smoothers.py:203-208): a smoother
    built outside a solver runs on its own one-level device context."""
    from paper_1902_01818_b200 import smoothers
    pr, setup, f, solver, orc = device_solver("cfg2", levels=3)
    A = solver.A[2]
    r = np.random.default_rng(8).standard_normal(A.shape[0])
    assert rel(smoothers.gs_apply_forward(A, r), orc.gs_forward(2, r)) <= 1e-12
    assert rel(smoothers.gs_apply_backward(A, r), orc.gs_backward(2, r)) <= 1e-12


@pytest.mark.parametrize("cfg,kw", [("cfg5", {"levels": 2}), ("cfg2", {"levels": 3})])
def test_matrix_free_operator_matches(cfg, kw):
    """Matrix-free finest operator (sum factorisation on affine conforming patches, mfree.cu),
    forced on small levels (IGB_MATRIX_FREE_MIN_NNZ=0): A x and f - A x against the assembled
    CSR to 1e-13, and the PCG solve against the oracle."""
    import os
    from paper_1902_01818_b200 import multigrid
    from oracle.solve import OracleSolver
    pr, setup, f = get_setup(cfg, **kw)
    os.environ["IGB_MATRIX_FREE_MIN_NNZ"] = "0"
    try:
        solver = multigrid.MultigridSolver(pr.hier, pr.config, device=0, setup=setup)
    finally:
        del os.environ["IGB_MATRIX_FREE_MIN_NNZ"]
    L = solver.finest
    A = solver.A[L]
    rng = np.random.default_rng(51)
    x, z = rng.standard_normal(A.shape[0]), rng.standard_normal(A.shape[0])
    y = solver.ctx.op("spmv", L, x, A.shape[0])
    assert rel(y, A @ x) <= 1e-13
    assert np.array_equal(solver.ctx.op("spmv", L, x, A.shape[0]), y)  # fixed order
    assert rel(solver.ctx.op("residual", L, x, A.shape[0], out_init=z), z - A @ x) <= 1e-13
    orc = OracleSolver(setup.setup_bundle())
    rep = solver.solve_pcg(f)
    xo, itso, histo = orc.solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
    assert rep.iterations == itso
    _check_history(rep.residuals, histo, f"{cfg} matrix-free vs oracle")
    assert rel(rep.x, xo) <= 1e-10
    solver.close()


def test_p6_backward_panel_far_slots_match_oracle():
    """cfg4 p = 6 (L = 4): backward rows carry up to 78 entries of another patch -- the panel
    variant with 5 far slots per lane (B = 512, several ranges); sweeps repeatable, equal to
    SuperLU on triu(A) per level."""
    pr, setup, f, solver, orc = device_solver("cfg4", p=6, levels=4)
    rng = np.random.default_rng(47)
    for level in range(1, solver.finest + 1):
        n = solver.A[level].shape[0]
        x = rng.standard_normal(n)
        for op, ref in (("gs_fwd", orc.gs_forward), ("gs_bwd", orc.gs_backward)):
            first = solver.ctx.op(op, level, x, n)
            for _ in range(3):
                assert np.array_equal(solver.ctx.op(op, level, x, n), first), (level, op)
            assert rel(first, ref(level, x)) <= 1e-12, (level, op)


def _solver_with_env(cfg, kw, env):
    import os
    from paper_1902_01818_b200 import multigrid
    pr, setup, f = get_setup(cfg, **kw)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        solver = multigrid.MultigridSolver(pr.hier, pr.config, device=0, setup=setup)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return pr, setup, f, solver


def test_kf10_panel_variant_is_opt_in():
    """The B = 256 / KF 10 panel variant (known wrong-result mode, DESIGN 9.2) never runs by default,
    IGB_PANEL_KF10=0 keeps it off, and IGB_PANEL_KF10=1 enables it on cfg4 p = 8's backward sweep."""
    pr, setup, f, solver = _solver_with_env("cfg4", {"p": 8, "levels": 3}, {})
    kfs = [solver.ctx.gs_info(l, d)["KF"] for l in range(1, 4) for d in (0, 1)]
    solver.close()
    assert 10 not in kfs
    pr, setup, f, solver = _solver_with_env("cfg4", {"p": 8, "levels": 3}, {"IGB_PANEL_KF10": "0"})
    assert 10 not in [solver.ctx.gs_info(l, d)["KF"] for l in range(1, 4) for d in (0, 1)]
    solver.close()
    # IGB_PANEL_HALF=2 lets every single-range B = 512 plan try the B = 256 alternative (at L = 3 the
    # default KA 14 trigger does not fire)
    pr, setup, f, solver = _solver_with_env("cfg4", {"p": 8, "levels": 3},
                                            {"IGB_PANEL_KF10": "1", "IGB_PANEL_HALF": "2"})
    info = solver.ctx.gs_info(3, 1)
    print(f"[kf10] cfg4 p=8 L=3 level 3 backward with IGB_PANEL_KF10=1: {info}")
    from oracle.solve import OracleSolver
    orc = OracleSolver(setup.setup_bundle())
    rng = np.random.default_rng(71)
    n = solver.A[3].shape[0]
    x = rng.standard_normal(n)
    first = solver.ctx.op("gs_bwd", 3, x, n)
    for _ in range(19):
        assert np.array_equal(solver.ctx.op("gs_bwd", 3, x, n), first)
    assert rel(first, orc.gs_backward(3, x)) <= 1e-12
    solver.close()


@pytest.mark.xfail(strict=True, reason="known defect of the opt-in B = 256 / KF 10 panel variant on a "
                   "single-range 3-D level (DESIGN 9.2): repeatable (20 bitwise-equal sweeps) but 7.6e-3 off "
                   "SuperLU; never planned by default (test_kf10_panel_variant_is_opt_in)")
def test_kf10_forced_on_3d_level():
    """IGB_PANEL_KF10_3D=1 forces the KF 10 panel variant onto cfg5 L = 2 (the level where DESIGN 9.2
    reproduced history drift): 20 repeated backward sweeps of every level bitwise identical and
    within 1e-12 of SuperLU, and the PCG history within 1e-10 per entry of the oracle."""
    pr, setup, f, solver = _solver_with_env("cfg5", {"levels": 2}, {"IGB_PANEL_KF10_3D": "1", "IGB_PANEL_HALF": "2"})
    from oracle.solve import OracleSolver
    orc = OracleSolver(setup.setup_bundle())
    infos = {(l, d): solver.ctx.gs_info(l, d) for l in (1, 2) for d in (0, 1)}
    print(f"[kf10-3d] {infos}")
    assert any(i["engine"] == "panel" and i["KF"] == 10 for i in infos.values()), "KF 10 not exercised"
    rng = np.random.default_rng(73)
    # the cycle's post-smoothing runs the sweep in accumulate mode (u += T^-1 r on matrix-free levels):
    # check one cycle first, then the plain sweeps
    r = rng.standard_normal(solver.n_dofs)
    print(f"[kf10-3d] cycle rel diff {rel(solver.cycle(2, r), orc.cycle(2, r)):.2e}")
    for level in (1, 2):
        n = solver.A[level].shape[0]
        x = rng.standard_normal(n)
        for op, ref in (("gs_fwd", orc.gs_forward), ("gs_bwd", orc.gs_backward)):
            first = solver.ctx.op(op, level, x, n)
            for _ in range(19):
                assert np.array_equal(solver.ctx.op(op, level, x, n), first), (level, op)
            assert rel(first, ref(level, x)) <= 1e-12, (level, op)
    rep = solver.solve_pcg(f, check_spd=False)
    xo, itso, histo = orc.solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
    assert rep.iterations == itso
    _check_history(rep.residuals, histo, "cfg5 L=2 KF 10 forced")
    solver.close()
