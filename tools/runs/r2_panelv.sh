export PYTHONUNBUFFERED=1
IGB_GS_DEBUG=1 IGB_VERBOSE=1 timeout 400 python tools/engine_check.py cfg5:levels=2 > gpurun_out/r2_panelv_L2.log 2>&1; echo "rc=$?" >> gpurun_out/r2_panelv_L2.log
timeout 900 python tools/fd3_check.py cfg5 --no-oracle --solves 2 2>&1 | tail -2 | cut -c1-260 > gpurun_out/r2_panelv_full.log
