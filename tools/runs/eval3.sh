timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "operators or flow" 2>&1 | tail -2
timeout 600 python tools/engine_compare.py cfg5:levels=3 "" "IGB_SPMV_GROUP=8" "IGB_FLOW_G=16"
timeout 600 python tools/engine_compare.py cfg2 "" "IGB_SPMV_GROUP=16"
timeout 1500 python tools/engine_compare.py cfg4:p=8 "" "IGB_GS_ENGINE=flow"
