export PYTHONUNBUFFERED=1 IGB_VERBOSE=1 IGB_GS_DEBUG=1 IGB_GS_ENGINE=wave
IGB_WAVE_RBMAX=500 timeout 600 python tools/engine_check.py cfg5:levels=3 > gpurun_out/r2_wave_L3_rb500.log 2>&1; echo "rc=$?" >> gpurun_out/r2_wave_L3_rb500.log
