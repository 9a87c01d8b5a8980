export PYTHONUNBUFFERED=1 IGB_PCG_GRAPH=0
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2_launches_plain.log 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2_launches_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2_launches_ncu.log
