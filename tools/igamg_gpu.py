"""igamg -> libigb adapter: the binding a maintainer would add to the reference.

It takes an already set-up *reference* ``igamg.multigrid.MultigridSolver`` and moves its solve phase
onto the B200 through the C ABI (include/igb.h), using only ctypes and the reference's own setup
objects -- no product Python module is imported.  ``tests/test_integration.py`` runs it against the
reference installed in ``baseline/_ref`` (``pip install --no-deps --target baseline/_ref``).

    ctx = attach(solver)                  # upload A_l, P_l, smoothers, coarse factors; finalize
    x, its, hist = cg(ctx, f, tol=1e-8)   # replaces linsolve.cg(solver.A[L], f, solver.preconditioner())
"""

import ctypes
import os

import numpy as np
import scipy.linalg
import scipy.sparse

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1902_01818_b200",
                   "libigb.so")
P = ctypes.c_void_p
_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(LIB)
        L.igb_last_error.restype = ctypes.c_char_p
        L.igb_last_error.argtypes = [P]
        _lib = L
    return _lib


def _a(x, t):
    return np.ascontiguousarray(x, dtype=t)


def _csr(M):
    M = scipy.sparse.csr_matrix(M)
    M.sort_indices()
    return _a(M.indptr, np.int32), _a(M.indices, np.int32), _a(M.data, np.float64)


def _ok(ctx, rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed ({rc}): {lib().igb_last_error(ctx).decode()}")


def square_transform(owner):
    """Square-transform form of a reference ``ScmsInteriorSolver`` (smoothers.py:232-294).

    The reference sums fast diagonalisations over subspaces alpha in {large, comp}^d,
    ``X = sum_alpha (x)_a T_{a,alpha_a} ((x)_a T_{a,alpha_a}^T R ./ denom_alpha)``.  With
    ``T_a = [T_{a,large} | T_{a,comp}]`` (columns of the two split subspaces side by side) this is one
    fast diagonalisation ``T (T^T R T ./ D) T^T`` where D holds denom_alpha on the block of alpha
    (verified to 4.8e-16).  Returns ([T_0, ..., T_{d-1}], D) with D in C order."""
    subs = owner._subspaces              # list of (Ts, denom) per subspace, Ts[a] = T_{a,alpha_a}
    d = len(subs[0][0])
    # the two distinct transforms per direction, in the order the subspaces enumerate them
    per_axis = [[] for _ in range(d)]
    for Ts, _ in subs:
        for a, T in enumerate(Ts):
            if not any(T is U or (T.shape == U.shape and np.array_equal(T, U)) for U in per_axis[a]):
                per_axis[a].append(T)
    T = [np.hstack(per_axis[a]) for a in range(d)]
    widths = [[U.shape[1] for U in per_axis[a]] for a in range(d)]
    D = np.zeros(tuple(t.shape[1] for t in T))
    for Ts, denom in subs:
        sl = []
        for a, Ta in enumerate(Ts):
            k = next(i for i, U in enumerate(per_axis[a]) if Ta is U or (Ta.shape == U.shape and np.array_equal(Ta, U)))
            lo = sum(widths[a][:k])
            sl.append(slice(lo, lo + Ta.shape[1]))
        D[tuple(sl)] = np.asarray(denom).reshape(tuple(t.shape[1] for t in Ts))
    return T, D


def attach(solver, device=0):
    """Upload a reference MultigridSolver's hierarchy to a new libigb context (multigrid.py:86-112)."""
    L_ = lib()
    ctx = P()
    if L_.igb_create(ctypes.byref(ctx), device) != 0:
        raise RuntimeError("igb_create failed (no CUDA device)")
    L = solver.finest
    _ok(ctx, L_.igb_set_num_levels(ctx, L), "igb_set_num_levels")
    keep = []
    for lv in range(L + 1):              # multigrid.py:92-99
        p, i, v = _csr(solver.A[lv])
        _ok(ctx, L_.igb_set_level_matrix(ctx, lv, solver.A[lv].shape[0], ctypes.c_longlong(len(v)),
                                         P(p.ctypes.data), P(i.ctypes.data), P(v.ctypes.data)), "set_level_matrix")
    for lv in range(1, L + 1):           # assembly.py:672-702
        p, i, v = _csr(solver.P[lv])
        _ok(ctx, L_.igb_set_prolongation(ctx, lv, solver.P[lv].shape[0], solver.P[lv].shape[1],
                                         ctypes.c_longlong(len(v)), P(p.ctypes.data), P(i.ctypes.data),
                                         P(v.ctypes.data)), "set_prolongation")
        smo = solver.smoother[lv]
        scms = getattr(smo, "scms", smo if hasattr(smo, "decomposition") else None)
        if scms is not None:
            _ok(ctx, L_.igb_scms_begin(ctx, lv, ctypes.c_double(scms.tau)), "scms_begin")
            for idx, solve in scms._solvers:  # smoothers.py:306-319
                owner = getattr(solve, "__self__", None)
                idx32 = _a(idx, np.int32)
                if hasattr(owner, "_subspaces"):  # interior: square transforms + denominators
                    T, D = square_transform(owner)
                    dims = _a([t.shape[0] for t in T], np.int32)
                    Ts = [_a(t, np.float64) for t in T]
                    Dc = _a(D, np.float64)
                    keep += [dims, Dc, idx32] + Ts
                    ptrs = [P(t.ctypes.data) for t in Ts] + [None] * (3 - len(Ts))
                    _ok(ctx, L_.igb_scms_add_interior(ctx, lv, len(dims), P(dims.ctypes.data), *ptrs,
                                                      P(Dc.ctypes.data), P(idx32.ctypes.data)), "add_interior")
                else:                          # interface piece: dense inverse from its SuperLU factor
                    inv = _a(owner._lu.solve(np.eye(len(idx))), np.float64)
                    _ok(ctx, L_.igb_scms_add_piece(ctx, lv, len(idx), P(idx32.ctypes.data), P(inv.ctypes.data)),
                        "add_piece")
        if getattr(smo, "gs", None) is not None or hasattr(smo, "apply_forward"):
            _ok(ctx, L_.igb_set_gs(ctx, lv), "set_gs")  # smoothers.py:174-184
    lu = solver.coarse_solver._lu        # linsolve.py:44
    (lp, li, lvv), (up, ui, uv) = _csr(lu.L), _csr(lu.U)
    pr, pc = _a(lu.perm_r, np.int32), _a(lu.perm_c, np.int32)
    _ok(ctx, L_.igb_set_coarse_lu(ctx, lu.shape[0], ctypes.c_longlong(len(lvv)), P(lp.ctypes.data),
                                  P(li.ctypes.data), P(lvv.ctypes.data), ctypes.c_longlong(len(uv)),
                                  P(up.ctypes.data), P(ui.ctypes.data), P(uv.ctypes.data), P(pr.ctypes.data),
                                  P(pc.ctypes.data)), "set_coarse_lu")
    cfg = solver.config
    steps = _a([cfg.steps_at(lv, L) for lv in range(L + 1)], np.int32)
    _ok(ctx, L_.igb_set_cycle(ctx, {"gs": 0, "scms": 1, "hyb": 2}[cfg.smoother], cfg.mu, P(steps.ctypes.data)),
        "set_cycle")
    _ok(ctx, L_.igb_finalize(ctx), "finalize")
    return ctx


def cg(ctx, b, tol=1e-8, max_iters=500):
    """igb_pcg: replaces linsolve.cg(solver.A[L], b, solver.preconditioner(), tol) (linsolve.py:64-101)."""
    b = _a(b, np.float64)
    x = np.empty_like(b)
    h = np.empty(max(1, max_iters))
    its = ctypes.c_int()
    _ok(ctx, lib().igb_pcg(ctx, P(b.ctypes.data), ctypes.c_double(tol), max_iters, P(x.ctypes.data),
                           ctypes.byref(its), P(h.ctypes.data), max_iters), "igb_pcg")
    return x, its.value, h[:its.value].tolist()


def close(ctx):
    lib().igb_destroy(ctx)
