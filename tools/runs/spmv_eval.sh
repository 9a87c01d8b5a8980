timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "operators or pcg_matches" 2>&1 | tail -2
timeout 600 python bench.py --config cfg5 --levels 3 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: (round(v['ms_per_step'],3), round(v['GBps'])) for k, v in d['roofline']['classes'].items()})"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: (round(v['ms_per_step'],3), round(v['GBps'])) for k, v in d['roofline']['classes'].items()})"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:spmv -c 400 --csv python bench.py --config cfg5 --levels 3 --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -v "^==" > gpurun_out/spmv_cfg5.csv
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/spmv_cfg5.csv")))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]; ik = h.index("Kernel Name"); im = h.index("Metric Name"); iv = h.index("Metric Value"); ig = h.index("Grid Size"); iid = h.index("ID")
per = {}
for r in rows[hi+1:]:
    if len(r) > iv: per.setdefault(r[iid], {"k": r[ik].split("(")[0][-22:] + r[ig]})[r[im]] = float(r[iv].replace(",", ""))
agg = collections.defaultdict(list)
for d in per.values(): agg[d["k"]].append((d.get("gpu__time_duration.sum", 0), d.get("dram__bytes_read.sum", 0)))
for k, v in agg.items():
    v.sort(); t, b = v[len(v)//2]
    print(k, len(v), "med us", t / 1e3, "dram MB", b / 1e6, "GB/s", b / t)
PY
