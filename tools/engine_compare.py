"""One host setup, several device solvers with different environment settings (GS engine,
flow parameters, ...): device PCG time per setting.

python tools/engine_compare.py cfg4:p=8 "IGB_GS_ENGINE=auto" "IGB_GS_ENGINE=flow" ...
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_01818_b200 import configs, multigrid  # noqa: E402

spec, *settings = sys.argv[1:]
name, *opts = spec.split(":")
t = time.perf_counter()
pr = configs.build(name, **{k: int(v) for k, v in (o.split("=") for o in opts)})
setup = multigrid.MultigridSetup(pr.hier, pr.config)
f = pr.rhs(setup.assembled_finest)
print(json.dumps({"cfg": spec, "N": setup.n_dofs, "setup_s": round(time.perf_counter() - t, 1)}), flush=True)
for st in settings or [""]:
    env = dict(kv.split("=", 1) for kv in st.split() if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    solver.ctx.pcg(f, pr.config.tol, pr.config.max_iters)
    ms = []
    for _ in range(3):
        x, its, hist = solver.ctx.pcg(f, pr.config.tol, pr.config.max_iters)
        ms.append(solver.ctx.last_timing()[0])
    print(json.dumps({"setting": st, "its": its, "device_ms": round(min(ms), 3), "final_rel": hist[-1]}), flush=True)
    solver.close()
