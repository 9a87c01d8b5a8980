"""Ablation timing of the panel sweep (IGB_GS_DEBUG cycles/panel on stderr).

python tools/panel_probe.py [cfg] [level]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["IGB_GS_DEBUG"] = "1"
from paper_1902_01818_b200 import configs, multigrid  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
pr = configs.build(spec)
setup = multigrid.MultigridSetup(pr.hier, pr.config)
lvl = int(sys.argv[2]) if len(sys.argv) > 2 else setup.finest
for pf in os.environ.get("PROBE_PF", "2").split(","):
    os.environ["IGB_PANEL_PF"] = pf
    solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
    n = solver.A[lvl].shape[0]
    x = np.random.default_rng(0).standard_normal(n)
    for ab in os.environ.get("PROBE_ABLATE", "0,1,2,4,8,16,3,7,31").split(","):
        os.environ["IGB_GS_ABLATE"] = ab
        print(f"pf {pf} ablate {ab}:", flush=True)
        for rep in range(2):
            solver.ctx.op("gs_fwd", lvl, x, n)
        sys.stderr.flush()
    solver.close()
