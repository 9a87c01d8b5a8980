"""One plain (non-graph) application of every hot-path kernel class on a configuration's finest
level, for `ncu --set full` (the PCG graph's conditional nodes cannot be profiled):

  spmv (matrix-free or CSR), gs_fwd, gs_bwd, scms (FD + interface pieces), restrict, prolong,
  then two iterations of unpreconditioned CG on the finest operator (dot, update, beta+direction).

python tools/ncu_ops.py cfg5 [--levels L]     prints the algorithmic bytes / flops of each op.
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
args = ap.parse_args()

from paper_1902_01818_b200 import configs, linsolve, multigrid  # noqa: E402

kw = {} if args.levels is None else {"levels": args.levels}
if args.p is not None:
    kw["p"] = args.p
pr = configs.build(args.config, **kw)
setup = multigrid.MultigridSetup(pr.hier, pr.config)
f = pr.rhs(setup.assembled_finest)
solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
ctx = solver.ctx
L = solver.finest
A = solver.A[L]
P = solver.P[L]
n, nc = A.shape[0], P.shape[1]
x = np.random.default_rng(5).standard_normal(n)
tri = (A.nnz - n) // 2
info = {
    "n": n, "nnz": int(A.nnz), "n_coarse": nc, "nnz_P": int(P.nnz),
    "alg_bytes": {
        "spmv_csr": 12 * A.nnz + 4 * (n + 1) + 16 * n,
        "gs_sweep": 12 * (tri + n) + 4 * (n + 1) + 24 * n,
        "restrict": 12 * P.nnz + 4 * (nc + 1) + 8 * n + 8 * nc,
        "prolong": 12 * P.nnz + 4 * (n + 1) + 8 * nc + 16 * n,
        "cg_update": 56 * n, "cg_beta_direction": 32 * n, "dot": 16 * n,
    },
    "gs_engines": [ctx.gs_info(L, d) for d in (0, 1)],
}
print(json.dumps(info), flush=True)
for op, m in (("spmv", n), ("gs_fwd", n), ("gs_bwd", n), ("scms", n), ("restrict", nc)):
    ctx.op(op, L, x, m)
ctx.op("prolong", L, np.ascontiguousarray(x[:nc]), n)
linsolve.cg(A, f, None, tol=1e-30, max_iters=2)
print("ops done", flush=True)
solver.close()
