export PYTHONUNBUFFERED=1 IGB_GS_DEBUG=1 IGB_VERBOSE=1
IGB_GS_ENGINE=panel timeout 600 python tools/engine_check.py cfg5:levels=3:nooracle > gpurun_out/r2_panel3.log 2>&1; echo "rc=$?" >> gpurun_out/r2_panel3.log
