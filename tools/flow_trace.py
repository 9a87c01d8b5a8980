"""Analyse an IGB_FLOW_TRACE dump of the dependency-driven sweep (flow.cu).

python tools/flow_trace.py DUMP.bin cfg[:key=val]
Per slot the kernel records [start time, crit seen - start, ready - crit seen, stored - ready
(cycles), stored time]; the matrix (rebuilt from the configuration) gives each row's last
dependency, so the hop from a dependency's store to the row's store can be decomposed.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

path, cfg = sys.argv[1], sys.argv[2]
upper = path.endswith("d1.bin")
raw = open(path, "rb").read()
nq = int(np.frombuffer(raw, np.int32, 1)[0])
row = np.frombuffer(raw, np.int32, nq, 4)
lev = np.frombuffer(raw, np.int32, nq, 4 + 4 * nq)
tr = np.frombuffer(raw, np.int64, 5 * nq, 4 + 8 * nq).reshape(nq, 5).astype(np.float64)
valid = row >= 0
t00 = tr[valid, 0].min()
tr[:, 0] -= t00
tr[:, 4] -= t00
L = int(lev.max()) + 1
done = np.array([tr[valid & (lev == l), 4].max() for l in range(L)])
d = np.diff(done)
print(f"slots {nq} levels {L} span {done[-1] / 1e3:.1f} us; per-level increment median {np.median(d):.0f} ns")
for i, name in ((1, "crit seen - start"), (2, "ready - crit seen"), (3, "stored - ready")):
    v = tr[valid, i]
    print(f"  {name:18s} cycles median {np.median(v):7.0f} p10 {np.percentile(v, 10):7.0f} p90 {np.percentile(v, 90):7.0f}")
from paper_1902_01818_b200 import configs, multigrid  # noqa: E402
name, *opts = cfg.split(":")
pr = configs.build(name, **{k: int(v) for k, v in (o.split("=") for o in opts)})
setup = multigrid.MultigridSetup(pr.hier, pr.config)
A = setup.A[int(path.split(".l")[1].split(".")[0])].tocsr()
qof = np.full(A.shape[0], -1)
qof[row[valid]] = np.nonzero(valid)[0]
gap, npend = [], []
for q in np.nonzero(valid)[0][nq // 3: nq // 3 + 4000]:
    i = row[q]
    c = A.indices[A.indptr[i]:A.indptr[i + 1]]
    c = c[c > i] if upper else c[c < i]
    if len(c) == 0:
        continue
    last = tr[qof[c], 4].max()
    gap.append(tr[q, 4] - last)
    npend.append(int((lev[qof[c]] == lev[q] - 1).sum()))
gap = np.array(gap)
print(f"stored - last dep stored: median {np.median(gap):.0f} ns p10 {np.percentile(gap, 10):.0f} "
      f"p90 {np.percentile(gap, 90):.0f}; deps one level back per row: median {np.median(npend):.0f}")
