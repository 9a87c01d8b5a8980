# default bench (cfg5 full) + reference arm, as the driver runs them
export PYTHONUNBUFFERED=1
( time timeout 1500 python bench.py --steps 20 --warmup 5 ) > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
( time timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r2_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench_ref.log
