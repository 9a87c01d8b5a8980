export PYTHONUNBUFFERED=1 IGB_GS_DEBUG=1 IGB_VERBOSE=1
for e in levels flow auto; do
  IGB_GS_ENGINE=$e timeout 400 python tools/engine_check.py cfg5:levels=2:nooracle > gpurun_out/r2_small_$e.log 2>&1; echo "rc=$?" >> gpurun_out/r2_small_$e.log
done
