export PYTHONUNBUFFERED=1
timeout 3000 python tools/large_run.py cfg1 cfg2 cfg3 cfg4:p=2:nooracle cfg4:p=4:nooracle cfg5:levels=3 cfg4:p=6:nooracle cfg4:p=8:nooracle 2> gpurun_out/r2_configs2.err | grep '^{' > gpurun_out/r2_configs2.jsonl
echo "rc=$?" >> gpurun_out/r2_configs2.err
