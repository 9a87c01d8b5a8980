import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1902_01818_b200 import configs, multigrid
pr = configs.build('cfg2')
setup = multigrid.MultigridSetup(pr.hier, pr.config)
solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
x = np.random.default_rng(0).standard_normal(solver.n_dofs)
for l in (5, 3):
    n = solver.A[l].shape[0]
    for rep in range(2):
        solver.ctx.op("gs_fwd", l, x[:n], n)
