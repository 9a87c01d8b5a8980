IGB_FLOW_TRACE=gpurun_out/tr_cfg5 timeout 300 python tools/gs_debug.py cfg5:levels=3 2>&1 | grep "flow level 3"
IGB_GS_ENGINE=flow IGB_FLOW_TRACE=gpurun_out/tr_cfg2 timeout 300 python tools/gs_debug.py cfg2 2>&1 | grep "flow level 5"
rm -f gpurun_out/tr_cfg5.l[12].* gpurun_out/tr_cfg2.l[1234].*
