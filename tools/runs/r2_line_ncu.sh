# ncu source-level capture of the line sweep (cfg5 L=3, level 3 forward = the 5th line launch)
export PYTHONUNBUFFERED=1
cat > /tmp/one_sweep.py <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np
from paper_1902_01818_b200 import configs, multigrid
pr=configs.build('cfg5', levels=3); s=multigrid.MultigridSetup(pr.hier, pr.config)
sv=multigrid.MultigridSolver(pr.hier, pr.config, setup=s)
n=s.A[3].shape[0]; x=np.random.default_rng(0).standard_normal(n)
for _ in range(2): sv.ctx.op('gs_fwd',3,x,n)
PY
IGB_GS_ENGINE=line timeout 600 ncu --set full --import-source on --clock-control none -k regex:line_sweep --launch-skip 1 -c 1 -o gpurun_out/r2_line_l3 -f python /tmp/one_sweep.py > gpurun_out/r2_line_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2_line_ncu.log
