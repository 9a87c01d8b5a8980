"""Check and time one Gauss-Seidel engine on a configuration.

  IGB_GS_ENGINE=line python tools/engine_check.py cfg5:levels=3 [cfg5 ...]

Per level and direction: the planned engine (igb_gs_info), 5 repeated sweeps bitwise equal,
relative difference to the oracle's sweep (C substitution, oracle/trisolve.c), and the device time
per sweep (CUDA events through IGB_GS_DEBUG, printed by the library); then the PCG solve time,
iteration count and history drift against the oracle's solve (skipped with :nooracle).
"""
import json
import os
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
    pr = configs.build(name, **kw)
    t = time.perf_counter()
    setup = multigrid.MultigridSetup(pr.hier, pr.config)
    f = pr.rhs(setup.assembled_finest)
    t_setup = time.perf_counter() - t
    t = time.perf_counter()
    solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
    t_up = time.perf_counter() - t
    from oracle.solve import OracleSolver
    orc = OracleSolver(setup.setup_bundle(), gs_impl="trisolve")
    rng = np.random.default_rng(5)
    out = {"cfg": spec, "engine": os.environ.get("IGB_GS_ENGINE", "auto"), "setup_s": round(t_setup, 1),
           "upload_s": round(t_up, 1), "levels": {}}
    for level in range(1, solver.finest + 1):
        n = solver.A[level].shape[0]
        x = rng.standard_normal(n)
        for d, (op, ref) in enumerate((("gs_fwd", orc.gs_forward), ("gs_bwd", orc.gs_backward))):
            info = solver.ctx.gs_info(level, d)
            first = solver.ctx.op(op, level, x, n)
            rep = all(np.array_equal(solver.ctx.op(op, level, x, n), first) for _ in range(4))
            r = ref(level, x)
            out["levels"][f"{level}.{d}"] = {"engine": info["engine"], "repeat_bitwise": rep,
                                             "rel": float(np.linalg.norm(first - r) / np.linalg.norm(r))}
            print(f"[check] level {level} {op}: {info} repeat {rep} rel {out['levels'][f'{level}.{d}']['rel']:.2e}",
                  flush=True)
    solver.ctx.pcg(f, pr.config.tol, pr.config.max_iters)
    x, its, hist = solver.ctx.pcg(f, pr.config.tol, pr.config.max_iters)
    out.update(its=its, device_ms=round(solver.ctx.last_timing()[0], 3))
    solver.ctx.profile(True)
    solver.ctx.profile_reset()
    solver.ctx.pcg(f, pr.config.tol, pr.config.max_iters)
    prof = solver.ctx.profile_get()
    solver.ctx.profile(False)
    out["classes_ms"] = {k: round(v["ms"], 3) for k, v in prof.items()}
    if with_oracle:
        xo, itso, histo = orc.solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
        h, ho = np.array(hist), np.array(histo)
        out.update(oracle_its=itso, hist_rel=float(np.max(np.abs(h - ho) / ho)) if len(h) == len(ho) else None,
                   x_rel=float(np.linalg.norm(x - xo) / np.linalg.norm(xo)))
    print(json.dumps(out), flush=True)
    solver.close()


if __name__ == "__main__":
    for s in sys.argv[1:]:
        run(s)
