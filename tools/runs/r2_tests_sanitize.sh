set -x
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q -s -p no:cacheprovider > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
for t in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize.py cfg2:3 > gpurun_out/r2_san_${t}_cfg2.log 2>&1; echo "rc=$?" >> gpurun_out/r2_san_${t}_cfg2.log
done
