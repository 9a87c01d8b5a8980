export PYTHONUNBUFFERED=1
timeout 900 python tools/fd3_check.py cfg5 --no-oracle > gpurun_out/r2_pf1_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pf1_full.log
timeout 600 python tools/fd3_check.py cfg5 --levels 3 > gpurun_out/r2_pf1_L3.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pf1_L3.log
IGB_FLOW_PREFETCH=0 timeout 600 python tools/fd3_check.py cfg5 --levels 3 --no-oracle > gpurun_out/r2_pf0_L3.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pf0_L3.log
