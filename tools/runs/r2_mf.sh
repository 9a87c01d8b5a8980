export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -q -p no:cacheprovider "tests/test_gpu_parity.py::test_matrix_free_operator_matches" "tests/test_gpu_parity.py::test_operators_match_oracle" > gpurun_out/r2_mf_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_mf_tests.log
timeout 900 python tools/fd3_check.py cfg5 --no-oracle --solves 2 2>&1 | tail -2 | cut -c1-400 > gpurun_out/r2_mf_full.log
