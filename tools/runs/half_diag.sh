# Diagnostic: B = 256 multi-range panel plans on every level that B = 512 runs as one range
O=gpurun_out
for kf in 1 0; do for c in cfg5:levels=2 cfg5:levels=3 cfg3 cfg2; do
  echo "== kf10=$kf $c"
  IGB_VERBOSE=1 IGB_PANEL_HALF=2 IGB_PANEL_KF10=$kf timeout 600 python tools/large_run.py $c 2>$O/half_err.log | tail -1 | cut -c1-400
  grep "panel sweep" $O/half_err.log | sed 's/inverse.*clusters/ clusters/'
done; done > $O/half_diag.log 2>&1
cat $O/half_diag.log | head -120
echo "== default cfg4:p=8" >> $O/half_diag.log
IGB_VERBOSE=1 timeout 900 python tools/large_run.py cfg4:p=8:nooracle 2>$O/half_err8.log | tail -1 | cut -c1-400 >> $O/half_diag.log
grep "panel\|flow" $O/half_err8.log | sed 's/inverse.*clusters/ clusters/' | head -20 >> $O/half_diag.log
tail -25 $O/half_diag.log
