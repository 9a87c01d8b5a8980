IGB_VERBOSE=1 timeout 600 python tools/plan_info.py cfg3 2>&1 | grep "panel sweep" | grep "level 4\|level 3"
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg3 or gs_sweeps" 2>&1 | tail -2
for c in cfg3 cfg2; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k, v in d['roofline']['classes'].items()})"; done
