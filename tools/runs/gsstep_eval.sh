timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --config cfg5 --levels 3 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: (round(v['ms_per_step'],3), round(v['GBps'])) for k, v in d['roofline']['classes'].items()})"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: (round(v['ms_per_step'],3), round(v['GBps'])) for k, v in d['roofline']['classes'].items()})"
for c in cfg3 cfg4:p=2; do timeout 600 python tools/engine_compare.py $c ""; done
