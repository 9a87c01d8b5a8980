# GPU suite (not the full-size module) with the per-case history drift printed
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -s -p no:cacheprovider > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
tail -5 gpurun_out/r2_pytest.log
