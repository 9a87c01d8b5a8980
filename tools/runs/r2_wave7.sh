export PYTHONUNBUFFERED=1 IGB_VERBOSE=1 IGB_GS_DEBUG=1 IGB_GS_ENGINE=wave
timeout 600 python tools/engine_check.py cfg5:levels=3 > gpurun_out/r2_wave_L3.log 2>&1; echo "rc=$?" >> gpurun_out/r2_wave_L3.log
IGB_WAVE_BACKOFF=0 IGB_WAVE_PBACKOFF=0 timeout 600 python tools/engine_check.py cfg5:levels=3 > gpurun_out/r2_wave_L3_nb.log 2>&1; echo "rc=$?" >> gpurun_out/r2_wave_L3_nb.log
IGB_WAVE_BACKOFF=1000 IGB_WAVE_PBACKOFF=100 timeout 600 python tools/engine_check.py cfg5:levels=3 > gpurun_out/r2_wave_L3_b512.log 2>&1; echo "rc=$?" >> gpurun_out/r2_wave_L3_b512.log
