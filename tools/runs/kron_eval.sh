timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for t in kron csr; do IGB_TRANSFER=$t timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', d['ms_per_step'], {k: round(v['ms_per_step'],3) for k, v in d['roofline']['classes'].items()})"; done
