timeout 600 ncu --kernel-name regex:"fd_|piece" --cache-control none --clock-control none --metrics gpu__time_duration.sum,launch__grid_size,sm__cycles_active.avg,smsp__inst_executed.sum --csv python tools/fd_probe.py cfg2 > gpurun_out/fd_ncu2.csv 2>gpurun_out/fd_ncu2.err
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/fd_ncu2.csv")))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]; ik = h.index("Kernel Name"); im = h.index("Metric Name"); iv = h.index("Metric Value"); iid = h.index("ID")
per = collections.OrderedDict()
for r in rows[hi+1:]:
    if len(r) <= iv: continue
    per.setdefault(r[iid], {"k": r[ik].split("(")[0][-22:]})[r[im]] = r[iv]
seen = collections.OrderedDict()
for d in per.values():
    key = (d["k"], d.get("launch__grid_size"))
    seen.setdefault(key, []).append((float(d.get("gpu__time_duration.sum", 0)), d.get("sm__cycles_active.avg"), d.get("smsp__inst_executed.sum")))
for k, v in seen.items():
    v.sort()
    print(k, len(v), "median us", v[len(v)//2][0] / 1e3, "cyc", v[len(v)//2][1], "inst", v[len(v)//2][2])
PY
