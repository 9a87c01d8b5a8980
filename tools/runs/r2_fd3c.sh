export PYTHONUNBUFFERED=1
timeout 600 python tools/fd3_check.py cfg5 --levels 3 > gpurun_out/r2_fd3c_L3.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fd3c_L3.log
timeout 900 python tools/fd3_check.py cfg5 --no-oracle > gpurun_out/r2_fd3c_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fd3c_full.log
IGB_FD3_BUF3=1 timeout 900 python tools/fd3_check.py cfg5 --levels 3 > gpurun_out/r2_fd3c_buf3_L3.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fd3c_buf3_L3.log
