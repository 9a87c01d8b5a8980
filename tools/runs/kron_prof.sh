for t in kron csr; do IGB_TRANSFER=$t timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', d['ms_per_step'], {k: round(v['ms_per_step'],3) for k, v in d['roofline']['classes'].items()})"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"kron|spmv_kernel" -c 400 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -v "^==" > gpurun_out/kron_launches.csv
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/kron_launches.csv")))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]; ik = h.index("Kernel Name"); iv = h.index("Metric Value"); ig = h.index("Grid Size") if "Grid Size" in h else None
agg = collections.defaultdict(list)
for r in rows[hi+1:]:
    if len(r) > iv: agg[(r[ik].split("(")[0][-40:], r[ig] if ig else "")].append(float(r[iv].replace(",", "")))
for k, v in sorted(agg.items()): print(k, len(v), "median ns", sorted(v)[len(v)//2])
PY
