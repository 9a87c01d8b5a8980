export PYTHONUNBUFFERED=1
timeout 600 python tools/fd3_check.py cfg5 --levels 3 > gpurun_out/r2_faces_L3.log 2>&1; echo "rc=$?" >> gpurun_out/r2_faces_L3.log
timeout 900 python -m pytest -q -p no:cacheprovider "tests/test_gpu_parity.py::test_operators_match_oracle" "tests/test_gpu_parity.py::test_pcg_matches_oracle_and_reference" "tests/test_gpu_parity.py::test_large_configs_match_reference_golden" "tests/test_gpu_parity.py::test_linsolve_cg_dropin_and_determinism" > gpurun_out/r2_faces_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_faces_tests.log
IGB_VERBOSE=1 timeout 900 python tools/fd3_check.py cfg5 --no-oracle > gpurun_out/r2_faces_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2_faces_full.log
