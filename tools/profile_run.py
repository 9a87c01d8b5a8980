"""Small fixed workload for ncu: build a config, run `--solves` PCG solves (device-resident).

python tools/profile_run.py [cfg2] [--levels L] [--solves 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="cfg2")
ap.add_argument("--levels", type=int, default=None)
ap.add_argument("--solves", type=int, default=2)
args = ap.parse_args()

from paper_1902_01818_b200 import configs, multigrid  # noqa: E402

kw = {} if args.levels is None else {"levels": args.levels}
pr = configs.build(args.config, **kw)
setup = multigrid.MultigridSetup(pr.hier, pr.config)
f = pr.rhs(setup.assembled_finest)
solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
ctx = solver.ctx
d_b = ctx.device_alloc(8 * len(f))
d_x = ctx.device_alloc(8 * len(f))
ctx.h2d(d_b, f)
for _ in range(args.solves):
    its, hist = ctx.pcg_device(d_b, d_x, pr.config.tol, pr.config.max_iters)
print("its", its, "ms", ctx.last_timing()[0], flush=True)
