# line engine: per-level timing (IGB_GS_DEBUG) on cfg5 L=3, parity check, full-size solve
export PYTHONUNBUFFERED=1
IGB_GS_ENGINE=line IGB_GS_DEBUG=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np
from paper_1902_01818_b200 import configs, multigrid
pr=configs.build('cfg5', levels=3); s=multigrid.MultigridSetup(pr.hier, pr.config)
sv=multigrid.MultigridSolver(pr.hier, pr.config, setup=s)
for l in range(1,4):
  n=s.A[l].shape[0]; x=np.random.default_rng(0).standard_normal(n)
  for op in ('gs_fwd','gs_bwd'):
    for _ in range(2): sv.ctx.op(op,l,x,n)
" > gpurun_out/r2_line_dbg.log 2>&1
IGB_GS_ENGINE=line timeout 600 python tools/engine_check.py cfg5:levels=3 > gpurun_out/r2_line_line.log 2>&1
IGB_GS_ENGINE=line timeout 900 python tools/engine_check.py cfg5:nooracle > gpurun_out/r2_line_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2_line_full.log
