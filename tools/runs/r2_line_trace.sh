export PYTHONUNBUFFERED=1
for lv in 1 2 3; do
IGB_GS_ENGINE=line timeout 600 python tools/line_trace.py cfg5:levels=3 $lv 0 >> gpurun_out/r2_line_trace.log 2>&1
done
IGB_GS_ENGINE=line timeout 600 python tools/engine_check.py cfg5:levels=3 > gpurun_out/r2_line_line.log 2>&1
