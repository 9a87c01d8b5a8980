for cfgv in "IGB_FLOW_CRITLAG=1" "IGB_FLOW_CRITLAG=2" "IGB_FLOW_CRITLAG=3" "IGB_FLOW_CRITLAG=2 IGB_FLOW_INFLIGHT=4" ; do
  echo "== $cfgv"
  env $cfgv timeout 300 python tools/gs_debug.py cfg5:levels=3 2>&1 | grep "flow level 3" | sed -n '2p;4p'
  env $cfgv IGB_GS_ENGINE=flow timeout 300 python tools/gs_debug.py cfg2 2>&1 | grep "flow level 5" | sed -n '2p;4p'
done
