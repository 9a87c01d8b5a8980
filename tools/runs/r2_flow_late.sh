# flow engine with the early/late split: per-level timing on cfg5 L=3 for several settings
export PYTHONUNBUFFERED=1
for cfgenv in "IGB_FLOW_LATE=32 IGB_FLOW_CRITLAG=4" "IGB_FLOW_LATE=48 IGB_FLOW_CRITLAG=5" "IGB_FLOW_LATE=64 IGB_FLOW_CRITLAG=6" "IGB_FLOW_LATE=64 IGB_FLOW_CRITLAG=8"; do
echo "== $cfgenv" >> gpurun_out/r2_flow_late.log
env $cfgenv IGB_GS_ENGINE=flow IGB_GS_DEBUG=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np
from paper_1902_01818_b200 import configs, multigrid
from oracle.solve import OracleSolver
pr=configs.build('cfg5', levels=3); s=multigrid.MultigridSetup(pr.hier, pr.config)
sv=multigrid.MultigridSolver(pr.hier, pr.config, setup=s)
orc=OracleSolver(s.setup_bundle(), gs_impl='trisolve')
for l in range(1,4):
  n=s.A[l].shape[0]; x=np.random.default_rng(0).standard_normal(n)
  for op,ref in (('gs_fwd',orc.gs_forward),('gs_bwd',orc.gs_backward)):
    for _ in range(2): y=sv.ctx.op(op,l,x,n)
    r=ref(l,x); print('rel',l,op,np.linalg.norm(y-r)/np.linalg.norm(r))
" >> gpurun_out/r2_flow_late.log 2>&1
done
grep -v "^\[igb\]" gpurun_out/r2_flow_late.log | grep "==\|us/level\|rel" | tail -80
