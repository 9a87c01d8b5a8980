export PYTHONUNBUFFERED=1 IGB_GS_DEBUG=1 IGB_FLOW_TRACE=gpurun_out/ftrace
timeout 900 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np
from paper_1902_01818_b200 import configs, multigrid
pr=configs.build('cfg5'); s=multigrid.MultigridSetup(pr.hier, pr.config)
sv=multigrid.MultigridSolver(pr.hier, pr.config, setup=s)
l=sv.finest; n=s.A[l].shape[0]; x=np.random.default_rng(0).standard_normal(n)
for op in ('gs_fwd','gs_bwd'):
    for _ in range(2): sv.ctx.op(op,l,x,n)
" > gpurun_out/r2_trace.log 2>&1
echo "rc=$?" >> gpurun_out/r2_trace.log
for d in 0 1; do python tools/flow_trace_quick.py gpurun_out/ftrace.l4.d$d.bin >> gpurun_out/r2_trace.log 2>&1; done
rm -f gpurun_out/ftrace.*.bin
