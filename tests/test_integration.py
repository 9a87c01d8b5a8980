"""The reference-side binding (tools/igamg_gpu.py) run on the reference itself.

The reference package is installed (unmodified, --no-deps) into baseline/_ref, which travels to the
GPU box; these tests skip when it is absent.

* CPU: ``square_transform`` applied to the reference's own ``ScmsInteriorSolver`` reproduces the
  reference's subspace-summed interior solve (smoothers.py:283-294) -- the identity the device FD
  relies on;
* GPU: ``attach`` uploads a reference ``MultigridSolver`` through the bare C ABI (no product Python
  module) and ``igb_pcg`` reproduces the reference's ``linsolve.cg(solver.A[L], f,
  solver.preconditioner(), tol=1e-8)``: identical iteration count, history within 1e-10 per entry,
  solution within 1e-10.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref")
pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "igamg")),
                                reason="reference not installed in baseline/_ref")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import igamg.assembly as ra
    import igamg.geometry as rg
    import igamg.linsolve as rl
    import igamg.multigrid as rm
    import igamg_gpu
    return ra, rg, rl, rm, igamg_gpu


def _solver(kind="hyb"):
    ra, rg, rl, rm, _ = _ref()
    hier = ra.build_hierarchy(rg.square_grid(2, 2), 3, 3, coarse_elements=4)
    solver = rm.MultigridSolver(hier, rm.CycleConfig(smoother=kind))
    f = ra.assemble_rhs(hier, solver.assembled_finest, ra.ManufacturedProblem(2))
    return solver, f


def test_square_transform_reproduces_reference_interior_solve():
    ra, rg, rl, rm, gpu = _ref()
    solver, f = _solver("scms")
    scms = solver.smoother[solver.finest]
    rng = np.random.default_rng(3)
    n_checked = 0
    for idx, solve in scms._solvers:
        owner = getattr(solve, "__self__", None)
        if not hasattr(owner, "_subspaces"):
            continue
        T, D = gpu.square_transform(owner)
        r = rng.standard_normal(len(idx))
        R = r.reshape(tuple(t.shape[0] for t in T))
        Y = R
        for a, Ta in enumerate(T):
            Y = np.moveaxis(np.tensordot(Ta.T, Y, axes=(1, a)), 0, a)
        Y = Y / D
        for a, Ta in enumerate(T):
            Y = np.moveaxis(np.tensordot(Ta, Y, axes=(1, a)), 0, a)
        ref = solve(r)
        assert np.linalg.norm(Y.ravel() - ref) <= 1e-13 * np.linalg.norm(ref)
        n_checked += 1
    assert n_checked > 0


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["hyb", "gs", "scms"])
def test_reference_solver_on_device_through_c_abi(kind):
    ra, rg, rl, rm, gpu = _ref()
    solver, f = _solver(kind)
    L = solver.finest
    x, its, hist = rl.cg(solver.A[L], f, solver.preconditioner(), tol=1e-8, max_iters=500)
    ctx = gpu.attach(solver)
    try:
        xd, itsd, histd = gpu.cg(ctx, f, tol=1e-8, max_iters=500)
    finally:
        gpu.close(ctx)
    assert itsd == its
    h, hd = np.array(hist), np.array(histd)
    assert np.max(np.abs(hd - h) / h) <= 1e-10
    assert np.linalg.norm(xd - x) <= 1e-10 * np.linalg.norm(x)
