timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "operators or pcg_matches or large_configs" 2>&1 | tail -1
timeout 600 python bench.py --config cfg5 --levels 3 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k, v in d['roofline']['classes'].items()})"
timeout 900 python tools/engine_compare.py cfg4:p=2 ""
