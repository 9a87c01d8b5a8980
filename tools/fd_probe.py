"""Per-level SCMS (fast diagonalisation + interface pieces) device time, via the profile API.

python tools/fd_probe.py [cfg[:key=val]]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_01818_b200 import configs, multigrid  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
name, *opts = spec.split(":")
pr = configs.build(name, **{k: int(v) for k, v in (o.split("=") for o in opts)})
setup = multigrid.MultigridSetup(pr.hier, pr.config)
solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
ctx = solver.ctx
rng = np.random.default_rng(0)
for l in range(solver.finest, 0, -1):
    smo = solver.smoother[l]
    scms = getattr(smo, "scms", None)
    if scms is None:
        continue
    n = solver.A[l].shape[0]
    x = rng.standard_normal(n)
    ints = [tuple(sol.dims) for _, sol in scms.interiors]
    for rep in range(3):
        ctx.op("scms", l, x, n)
    ctx.profile(True)
    ctx.profile_reset()
    reps = 20
    for rep in range(reps):
        ctx.op("scms", l, x, n)
    prof = ctx.profile_get()
    ctx.profile(False)
    fd = prof.get("fd", {})
    pc = prof.get("pieces", {})
    print(f"level {l}: n {n} interiors {len(ints)} {ints[:2]}.. pieces {len(scms.pieces)} fd {fd.get('ms', 0) / reps * 1e3:.1f} us "
          f"({fd.get('launches', 0) / reps:.0f} launches) pieces {pc.get('ms', 0) / reps * 1e3:.1f} us", flush=True)
