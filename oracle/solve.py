"""CPU oracle of the MG-PCG solve phase -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module, and
only as the checker / the timed CPU reference.  The product package
``paper_1902_01818_b200`` never imports it and has no CPU fallback.

It restates the reference's solve phase operation for operation with the same
third-party calls, so that on identical setup data it reproduces the
reference bit for bit (pinned in ``tests/test_oracle.py`` against the
reference itself and against ``tests/golden/*.npz``):

* ``cg``                         <- ``linsolve.cg``            (pkg/src/igamg/linsolve.py:64-101)
* ``OracleSolver.cycle``         <- ``MultigridSolver.cycle``  (multigrid.py:118-138)
* ``OracleSolver.check_spd``     <- ``check_preconditioner_spd`` (multigrid.py:144-159)
* ``_GaussSeidel``               <- ``smoothers.GaussSeidel``  (smoothers.py:171-200)
* ``_interior_solve``            <- ``ScmsInteriorSolver.solve`` (smoothers.py:283-294)
* ``_Scms.apply``                <- ``SubspaceCorrectedMass.apply`` (smoothers.py:321-325)
* hybrid pre/post smoothing      <- ``HybridSmoother``         (smoothers.py:343-353)
* ``OracleSolver.solve_stationary`` / ``solve_direct`` <- ``MultigridSolver._iterate`` with the
  stationary and line-search steps (multigrid.py:170-234)
* coarse / piece solves          <- ``linsolve.Factorization.solve`` (linsolve.py:33-53)
* ``_TriSolveGS``                 <- the same GS sweeps as row substitution in C
  (``oracle/trisolve.c``, built into ``oracle/_ref/libtrisolve.so``) for levels where
  ``splu(tril(A))`` does not fit (cfg4 p = 8, cfg5 at full size); equal to SuperLU to
  rounding, pinned against it in ``tests/test_oracle.py``.

Input is a *setup bundle* (plain dict: matrices ``A``, prolongations ``P``,
smoother kind, ``mu``, steps per level, per-level SCMS interior/piece data),
produced either by the product's host setup (``MultigridSetup.setup_bundle``)
or extracted from a reference ``MultigridSolver`` (``bundle_from_reference``).
"""

import ctypes
import os

import numpy as np
import scipy.sparse
import scipy.sparse.linalg

__all__ = ["cg", "OracleSolver", "bundle_from_reference", "trisolve_lib"]

_TRI_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "libtrisolve.so")
_tri = None
# levels with more strict-triangle entries than this use the C substitution (SuperLU's copy of
# tril(A) plus its supernodal workspace does not fit at cfg4 p = 8 / cfg5 full size)
SPLU_MAX_TRI_NNZ = int(os.environ.get("ORACLE_SPLU_MAX_TRI_NNZ", 60_000_000))


def trisolve_lib():
    """oracle/_ref/libtrisolve.so (built by oracle/Makefile via __graft_entry__.build())."""
    global _tri
    if _tri is None:
        if not os.path.exists(_TRI_LIB):
            import subprocess
            subprocess.run(["make", "-s", "-C", os.path.dirname(os.path.abspath(__file__))], check=True)
        lib = ctypes.CDLL(_TRI_LIB)
        for name in ("tri_forward", "tri_backward"):
            fn = getattr(lib, name)
            fn.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 5
            fn.restype = ctypes.c_int
        _tri = lib
    return _tri


def cg(A, b, preconditioner=None, tol=1e-8, max_iters=10000, callback=None):
    """PCG with recursive residual; returns (x, iterations, history) (linsolve.py:64-101)."""
    b = np.asarray(b, dtype=float)
    n = b.shape[0]
    normb = np.linalg.norm(b)
    x = np.zeros(n)
    if normb == 0.0:
        return x, 0, []
    apply_prec = preconditioner if preconditioner is not None else (lambda r: r)
    r = b.copy()
    z = apply_prec(r)
    d = z.copy()
    rz = r @ z
    history = []
    for it in range(1, max_iters + 1):
        Ad = A @ d
        alpha = rz / (d @ Ad)
        x += alpha * d
        r -= alpha * Ad
        rel = np.linalg.norm(r) / normb
        history.append(rel)
        if callback is not None:
            callback(it, rel)
        if rel <= tol:
            return x, it, history
        z = apply_prec(r)
        rz_new = r @ z
        beta = rz_new / rz
        rz = rz_new
        d = z + beta * d
    return x, max_iters, history


def _splu_spd(A):
    """SuperLU with SciPy defaults (COLAMD, partial pivoting) as linsolve.Factorization does."""
    return scipy.sparse.linalg.splu(scipy.sparse.csc_matrix(A))


class _GaussSeidel:
    def __init__(self, A):
        A = A.tocsr()
        if np.any(A.diagonal() == 0.0):
            raise ValueError("Gauss-Seidel needs a nonzero diagonal")
        tril = scipy.sparse.tril(A, format="csc")
        self._lu = scipy.sparse.linalg.splu(
            tril, permc_spec="NATURAL", diag_pivot_thresh=0.0, options={"SymmetricMode": True})

    def forward(self, r):
        return self._lu.solve(r, trans="N")

    def backward(self, r):
        return self._lu.solve(r, trans="T")


class _TriSolveGS:
    """Same sweeps as ``_GaussSeidel`` by row substitution on A's CSR (oracle/trisolve.c)."""

    def __init__(self, A):
        A = A.tocsr()
        if not A.has_sorted_indices:
            A = A.sorted_indices()
        if np.any(A.diagonal() == 0.0):
            raise ValueError("Gauss-Seidel needs a nonzero diagonal")
        self.n = A.shape[0]
        self.ptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
        self.col = np.ascontiguousarray(A.indices, dtype=np.int32)
        self.val = np.ascontiguousarray(A.data, dtype=np.float64)
        self.lib = trisolve_lib()

    def _run(self, fn, r):
        b = np.ascontiguousarray(r, dtype=np.float64)
        x = np.empty_like(b)
        rc = fn(self.n, self.ptr.ctypes.data, self.col.ctypes.data, self.val.ctypes.data, b.ctypes.data,
                x.ctypes.data)
        if rc != 0:
            raise ValueError("Gauss-Seidel needs a nonzero diagonal")
        return x

    def forward(self, r):
        return self._run(self.lib.tri_forward, r)

    def backward(self, r):
        return self._run(self.lib.tri_backward, r)


def make_gauss_seidel(A, impl="auto"):
    """SuperLU (bitwise the reference) unless the level is too large for splu(tril(A))."""
    if impl == "auto":
        impl = "superlu" if (A.nnz + A.shape[0]) // 2 <= SPLU_MAX_TRI_NNZ else "trisolve"
    return _GaussSeidel(A) if impl == "superlu" else _TriSolveGS(A)


def _interior_solve(subspaces, dims, r):
    R = np.asarray(r).reshape(dims)
    out = np.zeros_like(R)
    for Ts, denom in subspaces:
        Y = R
        for a, T in enumerate(Ts):
            Y = np.moveaxis(np.tensordot(T.T, Y, axes=(1, a)), 0, a)
        Y = Y / denom
        for a, T in enumerate(Ts):
            Y = np.moveaxis(np.tensordot(T, Y, axes=(1, a)), 0, a)
        out += Y
    return out.ravel()


class _Scms:
    def __init__(self, A, entry):
        self.tau = entry["tau"]
        self._solvers = []
        for it in entry["interiors"]:
            subs, dims = it["subspaces"], tuple(it["dims"])
            self._solvers.append((it["indices"], lambda r, s=subs, d=dims: _interior_solve(s, d, r)))
        A = A.tocsr()
        for idx in entry["pieces"]:
            lu = _splu_spd(A[idx][:, idx].tocsc())
            self._solvers.append((idx, lambda b, lu=lu: lu.solve(np.asarray(b, dtype=float), trans="N")))

    def apply(self, r):
        out = np.zeros_like(r)
        for indices, solve in self._solvers:
            out[indices] += solve(r[indices])
        return self.tau * out


class OracleSolver:
    """Reference-faithful cycle / preconditioner on a setup bundle."""

    def __init__(self, bundle, gs_impl="auto"):
        self.A = bundle["A"]
        self.P = bundle["P"]
        self.kind = bundle["smoother"]
        self.mu = bundle["mu"]
        self.steps = bundle["steps"]
        self.finest = bundle["finest"]
        self.coarse = _splu_spd(self.A[0])
        self.gs = [None] * (self.finest + 1)
        self.scms = [None] * (self.finest + 1)
        for level in range(1, self.finest + 1):
            if self.kind in ("gs", "hyb"):
                self.gs[level] = make_gauss_seidel(self.A[level], gs_impl)
            if self.kind in ("scms", "hyb"):
                self.scms[level] = _Scms(self.A[level], bundle["levels"][level])

    @property
    def n_dofs(self):
        return self.A[self.finest].shape[0]

    def _pre(self, level, A, u, f, steps):
        gs, scms = self.gs[level], self.scms[level]
        if self.kind == "gs":
            for _ in range(steps):
                u += gs.forward(f - A @ u)
        elif self.kind == "scms":
            for _ in range(steps):
                u += scms.apply(f - A @ u)
        else:
            u += gs.forward(f - A @ u)
            for _ in range(steps):
                u += scms.apply(f - A @ u)
        return u

    def _post(self, level, A, u, f, steps):
        gs, scms = self.gs[level], self.scms[level]
        if self.kind == "gs":
            for _ in range(steps):
                u += gs.backward(f - A @ u)
        elif self.kind == "scms":
            for _ in range(steps):
                u += scms.apply(f - A @ u)
        else:
            for _ in range(steps):
                u += scms.apply(f - A @ u)
            u += gs.backward(f - A @ u)
        return u

    def cycle(self, level, f, u=None):
        if level < 1:
            raise ValueError("cycles act on levels >= 1")
        A = self.A[level]
        u = np.zeros_like(f) if u is None else u
        steps = self.steps[level]
        u = self._pre(level, A, u, f, steps)
        r = self.P[level].T @ (f - A @ u)
        if level == 1:
            u = u + self.P[level] @ self.coarse.solve(np.asarray(r, dtype=float), trans="N")
        else:
            for _ in range(self.mu):
                correction = self.cycle(level - 1, r)
                u = u + self.P[level] @ correction
                if self.mu > 1:
                    r = self.P[level].T @ (f - A @ u)
        return self._post(level, A, u, f, steps)

    def preconditioner(self):
        return lambda r: self.cycle(self.finest, r)

    # single operators, for per-kernel parity tests
    def gs_forward(self, level, r):
        return self.gs[level].forward(r)

    def gs_backward(self, level, r):
        return self.gs[level].backward(r)

    def scms_apply(self, level, r):
        return self.scms[level].apply(r)

    def coarse_solve(self, r):
        return self.coarse.solve(np.asarray(r, dtype=float), trans="N")

    def check_spd(self, rtol=1e-8, seed=20240801):
        rng = np.random.default_rng(seed)
        r = rng.standard_normal(self.n_dofs)
        s = rng.standard_normal(self.n_dofs)
        Br, Bs = self.cycle(self.finest, r), self.cycle(self.finest, s)
        lhs, rhs = s @ Br, r @ Bs
        scale = max(abs(lhs), abs(rhs), 1e-30)
        return abs(lhs - rhs) <= rtol * scale and r @ Br > 0 and s @ Bs > 0

    def solve(self, b, tol=1e-8, max_iters=500):
        return cg(self.A[self.finest], b, self.preconditioner(), tol=tol, max_iters=max_iters)

    def _iterate(self, f, step, tol, max_iters):
        """(u, its, residuals, converged) of multigrid.py:170-200 (10 increases = divergence)."""
        normf = np.linalg.norm(f)
        u = np.zeros_like(f)
        if normf == 0.0:
            return u, 0, [], True
        residuals, increases = [], 0
        for it in range(1, max_iters + 1):
            u, rel = step(u)
            rel = rel / normf
            increases = increases + 1 if residuals and rel > residuals[-1] else 0
            residuals.append(rel)
            if rel <= tol:
                return u, it, residuals, True
            if increases >= 10 or not np.isfinite(rel):
                return u, it, residuals, False
        return u, max_iters, residuals, False

    def solve_stationary(self, f, tol=1e-8, max_iters=500):
        A = self.A[self.finest]

        def step(u):
            u = self.cycle(self.finest, f, u)
            return u, np.linalg.norm(f - A @ u)

        return self._iterate(f, step, tol, max_iters)

    def solve_direct(self, f, tol=1e-8, max_iters=500):
        A = self.A[self.finest]
        state = {"r": f.copy()}

        def step(u):
            r = state["r"]
            z = self.cycle(self.finest, r)
            Az = A @ z
            zAz = z @ Az
            if not np.isfinite(zAz) or zAz <= 0.0:
                return u, np.inf
            alpha = (r @ z) / zAz
            u = u + alpha * z
            state["r"] = r - alpha * Az
            return u, np.linalg.norm(state["r"])

        return self._iterate(f, step, tol, max_iters)


def bundle_from_reference(solver):
    """Setup bundle extracted from a *reference* ``igamg.multigrid.MultigridSolver``.

    Used only to pin the oracle against the reference in this container
    (SURVEY.md Appendix A "Adapter").
    """
    cfg = solver.config
    L = solver.finest
    levels = [None]
    for level in range(1, L + 1):
        smo = solver.smoother[level]
        scms = getattr(smo, "scms", None)
        if scms is None and hasattr(smo, "decomposition"):
            scms = smo
        entry = {}
        if scms is not None:
            entry["tau"] = scms.tau
            interiors, pieces = [], []
            for indices, solve in scms._solvers:
                owner = getattr(solve, "__self__", None)
                if owner is not None and hasattr(owner, "_subspaces"):
                    interiors.append({"indices": indices, "dims": owner.dims,
                                      "subspaces": owner._subspaces})
                else:
                    pieces.append(indices)
            entry["interiors"] = interiors
            entry["pieces"] = pieces
        levels.append(entry)
    return {
        "A": list(solver.A), "P": list(solver.P), "smoother": cfg.smoother, "mu": cfg.mu,
        "steps": [cfg.steps_at(l, L) for l in range(L + 1)], "levels": levels, "finest": L,
    }
