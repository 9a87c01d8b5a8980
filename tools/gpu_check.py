"""Per-operator device-vs-oracle shakedown (prints max relative differences).

python tools/gpu_check.py cfg1 cfg2:levels=3 ...
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1902_01818_b200 import configs, multigrid  # noqa: E402
from oracle.solve import OracleSolver  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def check(spec):
    name, *opts = spec.split(":")
    kw = {}
    for o in opts:
        k, v = o.split("=")
        kw[k] = int(v)
    t = time.perf_counter()
    pr = configs.build(name, **kw)
    setup = multigrid.MultigridSetup(pr.hier, pr.config)
    f = pr.rhs(setup.assembled_finest)
    t_setup = time.perf_counter() - t
    solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
    orc = OracleSolver(setup.setup_bundle())
    L = solver.finest
    rng = np.random.default_rng(1)
    out = {"cfg": spec, "N": solver.n_dofs, "setup_s": round(t_setup, 2)}
    ctx = solver.ctx
    for level in range(1, L + 1):
        n = solver.A[level].shape[0]
        x = rng.standard_normal(n)
        out[f"spmv{level}"] = rel(ctx.op("spmv", level, x, n), solver.A[level] @ x)
        if orc.gs[level] is not None:
            out[f"gsf{level}"] = rel(ctx.op("gs_fwd", level, x, n), orc.gs_forward(level, x))
            out[f"gsb{level}"] = rel(ctx.op("gs_bwd", level, x, n), orc.gs_backward(level, x))
        if orc.scms[level] is not None:
            out[f"scms{level}"] = rel(ctx.op("scms", level, x, n), orc.scms_apply(level, x))
        nc = solver.A[level - 1].shape[0]
        out[f"restr{level}"] = rel(ctx.op("restrict", level, x, nc), solver.P[level].T @ x)
        xc = rng.standard_normal(nc)
        out[f"prol{level}"] = rel(ctx.op("prolong", level, xc, n), solver.P[level] @ xc)
        out[f"cycle{level}"] = rel(ctx.op("cycle", level, x, n), orc.cycle(level, x))
    x0 = rng.standard_normal(solver.A[0].shape[0])
    out["coarse"] = rel(ctx.op("coarse", 0, x0, len(x0)), orc.coarse_solve(x0))
    rep = solver.solve_pcg(f)
    t = time.perf_counter()
    xo, itso, histo = orc.solve(f)
    t_cpu = time.perf_counter() - t
    h, ho = np.array(rep.residuals), np.array(histo)
    out.update(its=rep.iterations, its_oracle=itso,
               hist_rel=float(np.max(np.abs(h - ho) / ho)) if len(h) == len(ho) else None,
               x_rel=rel(rep.x, xo), device_ms=rep.device_ms, cpu_cg_s=round(t_cpu, 3))
    for k, v in out.items():
        if isinstance(v, float):
            out[k] = float(f"{v:.3e}")
    print(out, flush=True)
    solver.close()


if __name__ == "__main__":
    for spec in sys.argv[1:] or ["cfg1", "cfg2:levels=3"]:
        check(spec)
