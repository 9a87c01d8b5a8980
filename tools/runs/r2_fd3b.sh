export PYTHONUNBUFFERED=1
timeout 600 python tools/fd3_check.py cfg5 --levels 3 > gpurun_out/r2_fd3b_L3.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fd3b_L3.log
timeout 900 python tools/fd3_check.py cfg5 --no-oracle > gpurun_out/r2_fd3b_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fd3b_full.log
timeout 900 python tools/fd3_check.py cfg5 --no-oracle --ops 2 > gpurun_out/r2_fd3b_ops.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:fd3_kernel -c 3 -o gpurun_out/prof_fd3_r2b -f python tools/fd3_check.py cfg5 --no-oracle --ops 2 > gpurun_out/r2_fd3b_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2_fd3b_ncu.log
