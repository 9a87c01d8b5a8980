# the driver's GPU suite (all -m gpu tests, full-size module included), timed, with per-case output
export PYTHONUNBUFFERED=1
( time timeout 1700 python -m pytest tests -m gpu -q -s -p no:cacheprovider --durations=20 ) > gpurun_out/r2_gpusuite.log 2>&1
echo "rc=$?" >> gpurun_out/r2_gpusuite.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke.log
