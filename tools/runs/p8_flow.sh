timeout 1500 python tools/engine_compare.py cfg4:p=8 "" "IGB_FLOW_CRITLAG=3" "IGB_FLOW_CRITLAG=1" "IGB_FLOW_INFLIGHT=8" "IGB_FLOW_G=16"
