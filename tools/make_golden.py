"""Generate tests/golden/*.npz by running the REFERENCE (igamg) in this container.

Usage: python tools/make_golden.py [name ...]     (needs /root/reference; not run on the GPU box)

For every configuration the reference's own API builds the hierarchy exactly
as SURVEY.md 8(d) freezes it, runs
    x, its, hist = igamg.linsolve.cg(solver.A[L], f, solver.preconditioner(), tol=1e-8, max_iters=500)
and records: its, hist, x (full when N <= 100k, else norm + strided sample),
f, and setup fingerprints (per-level n / nnz / Frobenius norms, A_L @ v for
v = default_rng(0).standard_normal(N)).  It also checks that the oracle
(oracle/solve.py) run on the reference's setup reproduces the reference bit
for bit and stores that flag.
"""

import itertools
import os
import sys
import time

import numpy as np

REF = os.environ.get("IGAMG_REF", "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from igamg import assembly as ra, bspline as rb, geometry as rg, linsolve as rl, multigrid as rm  # noqa: E402

from oracle.solve import OracleSolver, bundle_from_reference  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def _sin_half(scale):
    def src(X):
        return scale * np.prod(np.sin(0.5 * np.pi * np.asarray(X)), axis=-1)
    return src


class _Src:
    """Source problem with g = 0 (reference assemble_rhs duck type)."""

    def __init__(self, f):
        self.f = f

    def source(self, X):
        return self.f(X) * np.ones(np.shape(X)[:-1])

    def dirichlet(self, X):
        return np.zeros(np.shape(X)[:-1])


def ref_cfg1(levels=3):
    dom = rg.unit_square()
    hier = ra.build_hierarchy(dom, 2, levels, "conforming", coarse_elements=8)
    return hier, rm.CycleConfig(smoother="scms", tau=1.0, delta=0.12), ra.ManufacturedProblem(2)


def ref_cfg2(levels=5):
    dom = rg.square_grid(2, 2)
    hier = ra.build_hierarchy(dom, 3, levels, coarse_elements=4)
    return hier, rm.CycleConfig(smoother="hyb"), _Src(_sin_half(2.0 * np.pi ** 2))


def ref_cfg3(levels=4):
    dom = rg.l_shape()
    hier = ra.DiscreteHierarchy(dom, 4, levels, "dg", "nonmatching")
    for lev in range(levels + 1):
        sp = [(rb.open_knot_vector(4, c, lev),) * 2 for c in (4, 8, 16)]
        hier.spaces.append(sp)
        hier.dofs.append(ra._build_dofs(dom, sp, "dg"))
    return (hier, rm.CycleConfig(smoother="hyb", tau=1.0, delta=0.12, sigma=5.0),
            _Src(lambda X: np.ones(np.shape(X)[:-1])))


def ref_cfg4(p=2, levels=6):
    dom = rg.distorted_grid(4, 4, 0.15, seed=1)
    hier = ra.build_hierarchy(dom, p, levels, coarse_elements=4)
    return hier, rm.CycleConfig(smoother="hyb"), _Src(_sin_half(1.0))


def ref_cfg5(levels=4):
    cubes = [rg._box_patch(o, np.asarray(o) + 1.0) for o in itertools.product((0.0, 1.0), repeat=3)]
    dom = rg.detect_interfaces(cubes)
    hier = ra.build_hierarchy(dom, 3, levels, coarse_elements=4)
    return hier, rm.CycleConfig(smoother="hyb"), ra.ManufacturedProblem(3)


CASES = {
    # name: (builder, kwargs, product-config name, product kwargs)
    "cfg1": (ref_cfg1, {}, "cfg1", {}),
    "cfg2": (ref_cfg2, {}, "cfg2", {}),
    "cfg3": (ref_cfg3, {}, "cfg3", {}),
    "cfg2_L3": (ref_cfg2, {"levels": 3}, "cfg2", {"levels": 3}),
    "cfg3_L2": (ref_cfg3, {"levels": 2}, "cfg3", {"levels": 2}),
    "cfg4_p2_L3": (ref_cfg4, {"p": 2, "levels": 3}, "cfg4", {"p": 2, "levels": 3}),
    "cfg4_p4_L3": (ref_cfg4, {"p": 4, "levels": 3}, "cfg4", {"p": 4, "levels": 3}),
    "cfg5_L1": (ref_cfg5, {"levels": 1}, "cfg5", {"levels": 1}),
    "cfg4_p2": (ref_cfg4, {"p": 2}, "cfg4", {"p": 2}),
    "cfg5_L2": (ref_cfg5, {"levels": 2}, "cfg5", {"levels": 2}),
    "cfg4_p8_L3": (ref_cfg4, {"p": 8, "levels": 3}, "cfg4", {"p": 8, "levels": 3}),
    "cfg4_p6_L3": (ref_cfg4, {"p": 6, "levels": 3}, "cfg4", {"p": 6, "levels": 3}),
    "cfg5_L3": (ref_cfg5, {"levels": 3}, "cfg5", {"levels": 3}),
    "cfg4_p4": (ref_cfg4, {"p": 4}, "cfg4", {"p": 4}),
}


def fingerprint(solver):
    L = solver.finest
    fp = {}
    fp["n"] = np.array([solver.A[l].shape[0] for l in range(L + 1)])
    fp["nnz"] = np.array([solver.A[l].nnz for l in range(L + 1)])
    fp["fro"] = np.array([np.sqrt((solver.A[l].data ** 2).sum()) for l in range(L + 1)])
    fp["p_nnz"] = np.array([0] + [solver.P[l].nnz for l in range(1, L + 1)])
    v = np.random.default_rng(0).standard_normal(solver.A[L].shape[0])
    fp["Av"] = solver.A[L] @ v
    return fp


def make(name):
    builder, kw, _, _ = CASES[name]
    t0 = time.perf_counter()
    hier, cfg, problem = builder(**kw)
    solver = rm.MultigridSolver(hier, cfg)
    f = ra.assemble_rhs(hier, solver.assembled_finest, problem)
    t_setup = time.perf_counter() - t0
    L = hier.L
    t1 = time.perf_counter()
    x, its, hist = rl.cg(solver.A[L], f, preconditioner=solver.preconditioner(), tol=cfg.tol,
                         max_iters=cfg.max_iters)
    t_cg = time.perf_counter() - t1
    oracle = OracleSolver(bundle_from_reference(solver))
    xo, itso, histo = oracle.solve(f, tol=cfg.tol, max_iters=cfg.max_iters)
    bitwise = bool(itso == its and np.array_equal(np.array(histo), np.array(hist)) and np.array_equal(xo, x))
    rng = np.random.default_rng(7)
    r = rng.standard_normal(len(f))
    cyc = solver.cycle(L, r.copy())
    fp = fingerprint(solver)
    N = len(f)
    data = dict(its=its, hist=np.array(hist), f=f, x_norm=np.linalg.norm(x),
                oracle_bitwise=bitwise, t_setup=t_setup, t_cg=t_cg, cycle_in_seed=7,
                **{f"fp_{k}": v for k, v in fp.items()})
    if N <= 100_000:
        data["x"] = x
        data["cycle_out"] = cyc
    else:
        step = max(1, N // 4096)
        data["x_sample_step"] = step
        data["x_sample"] = x[::step]
        data["cycle_sample"] = cyc[::step]
        data.pop("f")
        data["f_norm"] = np.linalg.norm(f)
        data["f_sample"] = f[::step]
        data["fp_Av"] = fp["Av"][::step]
        data["fp_Av_norm"] = np.linalg.norm(fp["Av"])
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **data)
    print(f"{name}: N={N} its={its} hist[-1]={hist[-1]:.3e} oracle_bitwise={bitwise} "
          f"setup={t_setup:.1f}s cg={t_cg:.2f}s", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or [n for n in CASES if n not in ("cfg4_p2", "cfg5_L3", "cfg4_p4")]
    for n in names:
        make(n)
