"""Per-row time budget of the flow sweep from an IGB_FLOW_TRACE dump (no matrix needed).

python tools/flow_trace_quick.py DUMP.bin
"""
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
nq = int(np.frombuffer(raw, np.int32, 1)[0])
row = np.frombuffer(raw, np.int32, nq, 4)
lev = np.frombuffer(raw, np.int32, nq, 4 + 4 * nq)
tr = np.frombuffer(raw, np.int64, 5 * nq, 4 + 8 * nq).reshape(nq, 5).astype(np.float64)
v = row >= 0
t0 = tr[v, 0].min()
span = tr[v, 4].max() - t0
L = int(lev.max()) + 1
print(f"rows {v.sum()} levels {L} span {span / 1e3:.1f} us = {span / L:.0f} ns per level, {v.sum() / L:.0f} rows per level")
dur = tr[v, 4] - tr[v, 0]
print(f"row start -> stored (ns): median {np.median(dur):.0f} p10 {np.percentile(dur, 10):.0f} p90 {np.percentile(dur, 90):.0f}")
for i, name in ((1, "start -> crit seen"), (2, "crit seen -> all values (early + late)"), (3, "values -> stored")):
    x = tr[v, i]
    print(f"  {name:40s} cycles median {np.median(x):7.0f} p10 {np.percentile(x, 10):7.0f} p90 {np.percentile(x, 90):7.0f}")
# lead: how long before its level's completion a row started
done = np.array([tr[v & (lev == l), 4].max() for l in range(L)])
lead = done[lev[v]] - tr[v, 0]
print(f"row start before its level is complete (ns): median {np.median(lead):.0f}")
