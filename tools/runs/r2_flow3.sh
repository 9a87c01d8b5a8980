export PYTHONUNBUFFERED=1
timeout 900 python tools/fd3_check.py cfg5 --no-oracle --solves 2 2>&1 | tail -2 | cut -c1-200 > gpurun_out/r2_flow3_full.log
timeout 600 python tools/fd3_check.py cfg5 --levels 3 --no-oracle 2>&1 | tail -2 | cut -c1-200 > gpurun_out/r2_flow3_L3.log
timeout 900 python -m pytest -q -p no:cacheprovider "tests/test_gpu_parity.py::test_flow_engine_matches_oracle" "tests/test_gpu_parity.py::test_pcg_matches_oracle_and_reference" > gpurun_out/r2_flow3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_flow3_tests.log
