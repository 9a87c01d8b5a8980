export PYTHONUNBUFFERED=1
timeout 900 python tools/fd3_check.py cfg5 --no-oracle --solves 2 2>&1 | tail -2 | cut -c1-260 > gpurun_out/r2_flow4_full.log
IGB_TRANSFER=kron timeout 900 python tools/fd3_check.py cfg5 --no-oracle --solves 2 2>&1 | tail -2 | cut -c1-360 > gpurun_out/r2_flow4_kron.log
timeout 900 python -m pytest -q -p no:cacheprovider "tests/test_gpu_parity.py::test_flow_engine_matches_oracle" "tests/test_fullsize.py::test_fullsize_pcg_matches_oracle" > gpurun_out/r2_flow4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_flow4_tests.log
