export PYTHONUNBUFFERED=1
timeout 900 python tools/ncu_ops.py cfg5 > gpurun_out/r2_ncu_ops_plain.log 2>&1 && \
timeout 2400 ncu --set full --clock-control none --import-source on \
  -k regex:'^(mf_|spmv_|piece_gemv|fd3_|flow_sweep|panel_sweep|cg_update|cg_beta|dot_kernel|kron_|copy_kernel)' -c 60 \
  -o gpurun_out/prof_ops_r2 -f python tools/ncu_ops.py cfg5 > gpurun_out/r2_ncu_ops.log 2>&1
echo "rc=$?" >> gpurun_out/r2_ncu_ops.log
