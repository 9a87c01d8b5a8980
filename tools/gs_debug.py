"""Per-sweep cycle counts of the device GS (IGB_GS_DEBUG=1) + parity vs SuperLU, per level.

python tools/gs_debug.py [cfg[:key=val]]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("IGB_GS_DEBUG", "1")
from paper_1902_01818_b200 import configs, multigrid  # noqa: E402
from oracle.solve import OracleSolver  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
name, *opts = spec.split(":")
pr = configs.build(name, **{k: int(v) for k, v in (o.split("=") for o in opts)})
setup = multigrid.MultigridSetup(pr.hier, pr.config)
solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
orc = OracleSolver(setup.setup_bundle())
rng = np.random.default_rng(0)
for l in range(solver.finest, 0, -1):
    if orc.gs[l] is None:
        continue
    n = solver.A[l].shape[0]
    x = rng.standard_normal(n)
    for op, ref in (("gs_fwd", orc.gs_forward), ("gs_bwd", orc.gs_backward)):
        for rep in range(2):
            y = solver.ctx.op(op, l, x, n)
        yr = ref(l, x)
        print(f"level {l} {op}: n {n} rel {np.linalg.norm(y - yr) / np.linalg.norm(yr):.3e}", flush=True)
