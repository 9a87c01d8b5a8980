export PYTHONUNBUFFERED=1
IGB_FLOW_CRITLAG=4 IGB_FLOW_LATE=32 timeout 1500 python tools/large_run.py cfg4:p=8:nooracle 2>/dev/null | grep '^{' | tail -1 > gpurun_out/r2_p8_lag4.json
