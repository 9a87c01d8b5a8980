timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "pcg or operators or cfg4_p2" 2>&1 | tail -2
for v in 0 1; do IGB_FD_LARGE=$v timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('large=$v', round(d['ms_per_step'],3), {k: (round(v['ms_per_step'],3), v['launches_per_step']) for k, v in d['roofline']['classes'].items()})"; done
for v in 0 1; do IGB_FD_LARGE=$v timeout 900 python tools/engine_compare.py cfg4:p=2 ""; done
