# Diagnostic: the B = 256 / KF 10 panel path forced onto 3-D levels (DESIGN 9.2)
O=gpurun_out
for env in "IGB_PANEL_KF10_3D=1" "IGB_PANEL_KF10_3D=1 IGB_PANEL_HALF=2" "IGB_PANEL_KF10_3D=1 IGB_PANEL_HALF=2 IGB_PANEL_KF10=0"; do
 for c in cfg5:levels=2 cfg5:levels=3; do
  echo "== $env $c"
  env $env IGB_VERBOSE=1 timeout 600 python tools/large_run.py $c 2>$O/k3_err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d.get(k) for k in ('its','oracle_its','device_ms','hist_rel_max','x_rel')})"
  grep "dir 1: panel\|dir 0: panel" $O/k3_err.log | sed 's/inverse.*clusters/ clusters/'
 done
done > $O/kf10_3d.log 2>&1
cat $O/kf10_3d.log
