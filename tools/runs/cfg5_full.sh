free -g | head -2
IGB_VERBOSE=1 timeout 3000 python tools/large_run.py cfg5:nooracle > gpurun_out/cfg5_full.log 2>&1
grep -v " fd\|fd plan" gpurun_out/cfg5_full.log | tail -12
