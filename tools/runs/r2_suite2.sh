export PYTHONUNBUFFERED=1
( time timeout 1200 python -m pytest tests/test_api_gpu.py tests/test_integration.py "tests/test_gpu_parity.py::test_linsolve_cg_dropin_and_determinism" "tests/test_gpu_parity.py::test_pinned_host_buffers_pcg_bitwise" "tests/test_gpu_parity.py::test_pcg_matches_oracle_and_reference" -m gpu -q -p no:cacheprovider ) > gpurun_out/r2_gpusuite2.log 2>&1
echo "rc=$?" >> gpurun_out/r2_gpusuite2.log
( time timeout 1500 python bench.py --steps 20 --warmup 5 ) > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
