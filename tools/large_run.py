"""Full-size runs: host setup, device PCG (timed), CPU oracle PCG (timed), parity summary.

python tools/large_run.py cfg5 [cfg4:p=8:nooracle ...]  ->  JSON lines per configuration
"""
import json
import os
import resource
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1902_01818_b200 import configs, multigrid  # noqa: E402


def run(spec):
    name, *opts = spec.split(":")
    with_oracle = "nooracle" not in opts
    opts = [o for o in opts if o != "nooracle"]
    kw = {k: int(v) for k, v in (o.split("=") for o in opts)}
    out = {"cfg": spec}
    t = time.perf_counter()
    pr = configs.build(name, **kw)
    setup = multigrid.MultigridSetup(pr.hier, pr.config)
    f = pr.rhs(setup.assembled_finest)
    out.update(N=setup.n_dofs, nnz=int(setup.A[setup.finest].nnz), setup_s=round(time.perf_counter() - t, 1),
               setup_phases={k: round(v, 1) for k, v in setup.timings.items()})
    t = time.perf_counter()
    solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
    out["upload_s"] = round(time.perf_counter() - t, 1)
    solver.ctx.pcg(f, pr.config.tol, pr.config.max_iters)  # warm-up (graph capture)
    x, its, hist = solver.ctx.pcg(f, pr.config.tol, pr.config.max_iters)
    dev_ms = solver.ctx.last_timing()[0]
    out.update(its=its, device_ms=round(dev_ms, 2), dofit_per_s=setup.n_dofs * its / (dev_ms / 1e3),
               final_rel=hist[-1])
    print(json.dumps(out), flush=True)
    if with_oracle:
        from oracle.solve import OracleSolver
        t = time.perf_counter()
        orc = OracleSolver(setup.setup_bundle())
        t1 = time.perf_counter()
        xo, itso, histo = orc.solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
        t2 = time.perf_counter()
        h, ho = np.array(hist), np.array(histo)
        out.update(oracle_its=itso, oracle_setup_s=round(t1 - t, 1), oracle_cg_s=round(t2 - t1, 2),
                   oracle_threads=os.environ.get("OMP_NUM_THREADS", "default"),
                   hist_rel_max=float(np.max(np.abs(h - ho) / ho)) if len(h) == len(ho) else None,
                   hist_rel_h1=float(np.max(np.abs(h - ho)) / ho[0]) if len(h) == len(ho) else None,
                   x_rel=float(np.linalg.norm(x - xo) / np.linalg.norm(xo)),
                   speedup_vs_oracle=round((t2 - t1) / (dev_ms / 1e3), 1))
    out["maxrss_gb"] = round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 1)
    print(json.dumps(out), flush=True)
    solver.close()


if __name__ == "__main__":
    for spec in sys.argv[1:] or ["cfg5"]:
        run(spec)
