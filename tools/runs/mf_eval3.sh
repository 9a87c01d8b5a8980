timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "matrix_free or large_configs or pcg_matches or operators" 2>&1 | tail -2
timeout 600 python bench.py --config cfg5 --levels 3 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: (round(v['ms_per_step'],3), round(v['GBps'])) for k, v in d['roofline']['classes'].items()})"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', round(d['ms_per_step'],3))"
timeout 1500 python tools/large_run.py cfg5:nooracle 2>&1 | tail -1
