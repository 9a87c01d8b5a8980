export PYTHONUNBUFFERED=1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/dmma_probe.cu -o /tmp/dmma_probe.bin && timeout 120 /tmp/dmma_probe.bin > gpurun_out/r2_dmma_probe.log 2>&1
for L in 2 3; do
  timeout 600 python tools/fd3_check.py cfg5 --levels $L > gpurun_out/r2_fd3_L$L.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fd3_L$L.log
  IGB_FD3=0 timeout 600 python tools/fd3_check.py cfg5 --levels $L --no-oracle > gpurun_out/r2_fd3off_L$L.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fd3off_L$L.log
done
timeout 900 python tools/fd3_check.py cfg5 --no-oracle > gpurun_out/r2_fd3_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fd3_full.log
