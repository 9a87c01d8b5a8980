timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "pinned or linsolve or zero_rhs or pcg_matches" 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['value'], d['e2e'])"
