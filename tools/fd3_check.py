"""FD check: SCMS operator of every level against the oracle, then per-class profile of PCG solves.

python tools/fd3_check.py cfg5 [--levels L] [--solves 3]     (IGB_FD3=0 selects the batched-GEMM path)
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="cfg5")
ap.add_argument("--levels", type=int, default=None)
ap.add_argument("--p", type=int, default=None)
ap.add_argument("--solves", type=int, default=3)
ap.add_argument("--no-oracle", action="store_true")
ap.add_argument("--ops", type=int, default=0, help="plain (non-graph) SCMS applications on the finest level, for ncu")
args = ap.parse_args()

from paper_1902_01818_b200 import configs, multigrid  # noqa: E402

kw = {} if args.levels is None else {"levels": args.levels}
if args.p is not None:
    kw["p"] = args.p
pr = configs.build(args.config, **kw)
setup = multigrid.MultigridSetup(pr.hier, pr.config)
f = pr.rhs(setup.assembled_finest)
solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
ctx = solver.ctx
if not args.no_oracle:
    from oracle.solve import OracleSolver
    orc = OracleSolver(setup.setup_bundle())
    rng = np.random.default_rng(5)
    for level in range(1, solver.finest + 1):
        if orc.scms[level] is None:
            continue
        n = solver.A[level].shape[0]
        x = rng.standard_normal(n)
        a = ctx.op("scms", level, x, n)
        b = orc.scms_apply(level, x)
        print(f"level {level} n {n}: scms rel diff {np.linalg.norm(a - b) / np.linalg.norm(b):.2e}", flush=True)
if args.ops:
    xr = np.random.default_rng(5).standard_normal(len(f))
    for _ in range(args.ops):
        ctx.op("scms", solver.finest, xr, len(f))
    print("ops done", flush=True)
    solver.close()
    sys.exit(0)
d_b = ctx.device_alloc(8 * len(f))
d_x = ctx.device_alloc(8 * len(f))
ctx.h2d(d_b, f)
for _ in range(2):
    its, hist = ctx.pcg_device(d_b, d_x, pr.config.tol, pr.config.max_iters)
print("its", its, "ms", ctx.last_timing()[0], "final", hist[-1], flush=True)
ctx.profile(True)
ctx.profile_reset()
for _ in range(args.solves):
    ctx.pcg_device(d_b, d_x, pr.config.tol, pr.config.max_iters)
prof = ctx.profile_get()
ctx.profile(False)
print(json.dumps({k: {"ms_per_solve": round(v["ms"] / args.solves, 3), "launches": v["launches"] / args.solves}
                  for k, v in prof.items()}), flush=True)
solver.close()
