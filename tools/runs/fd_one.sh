timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "operators or pcg or smoother" 2>&1 | tail -2
for v in 0 20 40 70; do IGB_FD_ONE_NMAX=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('one<=$v', round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k, v in d['roofline']['classes'].items()})"; done
for v in 0 40; do IGB_FD_ONE_NMAX=$v timeout 600 python tools/engine_compare.py cfg3 ""; done
