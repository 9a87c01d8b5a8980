"""Drive every hot-path kernel family once under compute-sanitizer (memcheck / racecheck / synccheck).

  compute-sanitizer --tool racecheck python tools/sanitize.py cfg2:3 cfg5:2 cfg4p8:3

Per configuration: each level's forward / backward Gauss-Seidel sweep (panel, flow or level-set
engine as planned), the SCMS apply (FD front/back or batched GEMM + interface pieces), SpMV,
residual, restriction / prolongation, the coarse solve, one cycle and one PCG solve (CUDA graph).
Optional env flags are passed through (e.g. IGB_PANEL_KF10_3D=1, IGB_GS_ENGINE=flow).
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(spec):
    from paper_1902_01818_b200 import configs, multigrid
    name, lv = spec.split(":")
    kw = {"levels": int(lv)}
    if name.startswith("cfg4p"):
        kw["p"] = int(name[5:])
        name = "cfg4"
    pr = configs.build(name, **kw)
    setup = multigrid.MultigridSetup(pr.hier, pr.config)
    f = pr.rhs(setup.assembled_finest)
    solver = multigrid.MultigridSolver(pr.hier, pr.config, device=0, setup=setup)
    ctx = solver.ctx
    rng = np.random.default_rng(1)
    for level in range(1, solver.finest + 1):
        n, nc = solver.A[level].shape[0], solver.A[level - 1].shape[0]
        x = rng.standard_normal(n)
        for d in (0, 1):
            print(f"[sanitize] {spec} level {level} dir {d}: {ctx.gs_info(level, d)}", flush=True)
        for op in ("spmv", "gs_fwd", "gs_bwd", "scms", "cycle"):
            ctx.op(op, level, x, n)
        ctx.op("residual", level, x, n, out_init=x)
        ctx.op("restrict", level, x, nc)
        ctx.op("prolong", level, rng.standard_normal(nc), n)
    ctx.op("coarse", 0, rng.standard_normal(solver.A[0].shape[0]), solver.A[0].shape[0])
    rep = solver.solve_pcg(f, check_spd=False)
    print(f"[sanitize] {spec}: pcg its {rep.iterations} final {rep.final_residual:.3e}", flush=True)
    solver.close()


if __name__ == "__main__":
    for s in sys.argv[1:] or ["cfg2:3"]:
        run(s)
    print("[sanitize] done", flush=True)
