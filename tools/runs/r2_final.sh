export PYTHONUNBUFFERED=1
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 ) > gpurun_out/r2_gpusuite.log 2>&1
echo "rc=$?" >> gpurun_out/r2_gpusuite.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke.log
( time timeout 1500 python bench.py --steps 20 --warmup 5 ) > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
( time timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r2_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench_ref.log
