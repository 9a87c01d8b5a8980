timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "flow or gs_sweeps" 2>&1 | tail -3
timeout 600 python bench.py --config cfg5 --levels 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5L3.log 2>&1; tail -1 gpurun_out/bench_cfg5L3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value']); [print(k, v) for k, v in d['roofline']['classes'].items()]"
IGB_VERBOSE=1 timeout 1500 python tools/large_run.py cfg4:p=8:nooracle > gpurun_out/cfg4p8.log 2>&1; grep -v "fd\b" gpurun_out/cfg4p8.log | grep "level 6\|cfg" | tail -8
