"""Critical-path analysis of one line sweep (line.cu) from its per-position trace.

  IGB_GS_ENGINE=line python tools/line_trace.py cfg5:levels=3 3 [0|1]

Runs the level's sweep with IGB_GS_DEBUG=1 IGB_LINE_TRACE (publish globaltimer, D / C poll
cycles per position), then for every position finds the dependency published last and the delay
from it to the position's own publish, classified by edge type (own line / same bundle / other
bundle), and walks the critical path back from the last position.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(spec, level, direction):
    path = "/tmp/line_trace"
    os.environ["IGB_GS_DEBUG"] = "1"
    os.environ["IGB_LINE_TRACE"] = path
    os.environ.setdefault("IGB_GS_ENGINE", "line")
    from paper_1902_01818_b200 import configs, multigrid
    name, *opts = spec.split(":")
    kw = {k: int(v) for k, v in (o.split("=") for o in opts)}
    pr = configs.build(name, **kw)
    setup = multigrid.MultigridSetup(pr.hier, pr.config)
    solver = multigrid.MultigridSolver(pr.hier, pr.config, setup=setup)
    A = setup.A[level].tocsr()
    n = A.shape[0]
    x = np.random.default_rng(0).standard_normal(n)
    op = "gs_bwd" if direction else "gs_fwd"
    for _ in range(3):
        solver.ctx.op(op, level, x, n)
    raw = open(f"{path}.l{level}.d{direction}.bin", "rb").read()
    hdr = np.frombuffer(raw[:12], dtype=np.int32)
    n_, nl, nb = (int(v) for v in hdr)
    off = 12
    lstart = np.frombuffer(raw[off:off + 4 * (nl + 1)], dtype=np.int32)
    off += 4 * (nl + 1)
    bstart = np.frombuffer(raw[off:off + 4 * (nb + 1)], dtype=np.int32)
    off += 4 * (nb + 1)
    tr = np.frombuffer(raw[off:], dtype=np.int64).reshape(n, 3)
    t = tr[:, 0].astype(np.float64)
    t -= t.min()
    line = np.searchsorted(lstart, np.arange(n), side="right") - 1
    bund = np.searchsorted(bstart, np.arange(n), side="right") - 1
    # position-space dependencies
    rows = np.arange(n)
    pos_of_row = (n - 1 - rows) if direction else rows
    crit = np.full(n, -1)
    for r in range(n):
        p = pos_of_row[r]
        cols = A.indices[A.indptr[r]:A.indptr[r + 1]]
        q = pos_of_row[cols]
        q = q[q < p]
        if len(q):
            crit[p] = q[np.argmax(t[q])]
    kinds = {0: "own line", 1: "same bundle", 2: "other bundle"}
    has = crit >= 0
    pp = np.flatnonzero(has)
    qq = crit[has]
    kind = np.where(line[pp] == line[qq], 0, np.where(bund[pp] == bund[qq], 1, 2))
    delay = t[pp] - t[qq]
    print(f"{spec} level {level} dir {direction}: n {n} lines {nl} bundles {nb} sweep {t.max() / 1e3:.1f} us")
    for k, name_ in kinds.items():
        m = kind == k
        if m.any():
            print(f"  last dependency {name_:13s}: {m.sum():7d} positions, delay median {np.median(delay[m]):7.0f} ns, "
                  f"p90 {np.percentile(delay[m], 90):7.0f} ns")
    # walk the critical path back from the last publish
    p = int(np.argmax(t))
    path_k, path_d = [], []
    while crit[p] >= 0:
        q = crit[p]
        path_k.append(0 if line[p] == line[q] else (1 if bund[p] == bund[q] else 2))
        path_d.append(t[p] - t[q])
        p = q
    path_k, path_d = np.array(path_k), np.array(path_d)
    print(f"  critical path: {len(path_k)} edges, {path_d.sum() / 1e3:.1f} us; start at {t[p] / 1e3:.1f} us")
    for k, name_ in kinds.items():
        m = path_k == k
        if m.any():
            print(f"    {name_:13s}: {m.sum():6d} edges, mean {path_d[m].mean():7.0f} ns, total {path_d[m].sum() / 1e3:8.1f} us")
    print(f"  D poll cycles: median {np.median(tr[:, 1]):.0f}, C poll cycles (rows that polled): "
          f"median {np.median(tr[tr[:, 2] > 0, 2]) if (tr[:, 2] > 0).any() else 0:.0f}, "
          f"fraction polled {np.mean(tr[:, 2] > 0):.2f}")
    solver.close()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 0)
