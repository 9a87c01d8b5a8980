# Diagnostic: 3-D KF 10 panel sweep with every far slot loaded (IGB_PANEL_ALLSLOTS) vs per-panel slot counts
O=gpurun_out
for env in "IGB_PANEL_KF10_3D=1 IGB_PANEL_ALLSLOTS=1" "IGB_PANEL_KF10_3D=1"; do
  echo "== $env cfg5:levels=2"
  env $env timeout 600 python tools/large_run.py cfg5:levels=2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d.get(k) for k in ('its','oracle_its','device_ms','hist_rel_max','x_rel')})"
done > $O/kf10_slots.log 2>&1
cat $O/kf10_slots.log
