export PYTHONUNBUFFERED=1
for v in "IGB_FLOW_WIDE_INFLIGHT=100" "IGB_FLOW_WIDE_INFLIGHT=1000" "IGB_FLOW_WIDE_INFLIGHT=14 IGB_FLOW_WIDE_LAG=3 IGB_FLOW_WIDE_LATE=16"; do
  echo "== $v" >> gpurun_out/r2_thr.log
  env $v timeout 900 python tools/fd3_check.py cfg5 --no-oracle --solves 2 2>&1 | tail -2 | cut -c1-200 >> gpurun_out/r2_thr.log
done
