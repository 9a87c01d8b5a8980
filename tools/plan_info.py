"""Print the sweep plans chosen for a configuration (IGB_VERBOSE=1) and time one GS op per level."""
import os, sys, time
os.environ.setdefault("IGB_VERBOSE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1902_01818_b200 import configs, multigrid
name, *opts = (sys.argv[1] if len(sys.argv) > 1 else "cfg2").split(":")
kw = {k: int(v) for k, v in (o.split("=") for o in opts)}
pr = configs.build(name, **kw)
setup = multigrid.MultigridSetup(pr.hier, pr.config)
solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
x = np.random.default_rng(0).standard_normal(solver.n_dofs)
for l in range(solver.finest, 0, -1):
    n = solver.A[l].shape[0]
    solver.ctx.op("gs_fwd", l, x[:n], n)
    t = time.perf_counter()
    for _ in range(3):
        solver.ctx.op("gs_fwd", l, x[:n], n)
    print(f"level {l}: gs_fwd op {(time.perf_counter() - t) / 3 * 1e3:.2f} ms (incl. H2D/D2H)", flush=True)
