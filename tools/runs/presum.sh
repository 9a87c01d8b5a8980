timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "gs_sweeps or pcg_matches or p8 or flow or cluster" 2>&1 | tail -2
IGB_GS_DEBUG=1 timeout 300 python tools/gs_debug.py cfg2 2>&1 | grep "panel level 5\|panel level 4" | sed -n '2p;4p;6p;8p'
for c in cfg2 cfg3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k, v in d['roofline']['classes'].items()})"; done
