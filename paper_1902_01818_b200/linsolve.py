"""Linear-algebra plumbing: host factorizations (setup) and the device PCG.

Mirrors ``igamg.linsolve`` (``linsolve.py:14-21``):

* :class:`Factorization` / :func:`factorize` -- SuperLU factorization on the
  host, exactly as the reference builds it (``linsolve.py:33-46``).  It is setup:
  the device consumes its ``L``, ``U``, ``perm_r``, ``perm_c`` (coarse solve) or
  the dense inverse built from it (interface pieces).
* :func:`cg` -- the reference's PCG semantics (x0 = 0, recursive residual, stop
  at ``||r||/||b|| <= tol``, history of relative residuals, ``(x, its, history)``
  with ``its = max_iters`` and the full history on non-convergence,
  ``linsolve.py:64-101``) executed entirely on the device when the
  preconditioner is a :class:`~paper_1902_01818_b200.multigrid.DevicePreconditioner`.
"""

import numpy as np
import scipy.sparse
import scipy.sparse.linalg

__all__ = ["Factorization", "factorize", "solve", "cg", "dense_generalized_eig", "write_coo", "read_coo",
           "DEFAULT_TOL"]

DEFAULT_TOL = 1e-8


class Factorization:
    """SuperLU factorization of a square sparse matrix (host setup)."""

    def __init__(self, A, spd=False):
        A = scipy.sparse.csc_matrix(A)
        if A.shape[0] != A.shape[1]:
            raise ValueError("matrix must be square")
        if spd:
            asym = abs(A - A.T)
            if asym.nnz and asym.max() > 1e-10 * max(1.0, abs(A).max()):
                raise ValueError("SPD factorization requested for unsymmetric matrix")
        self.shape = A.shape
        self.spd = spd
        try:
            self._lu = scipy.sparse.linalg.splu(A)
        except RuntimeError as exc:
            raise ValueError(f"matrix is numerically singular: {exc}") from exc

    def factors(self):
        """(L csr with unit diagonal, U csr, perm_r, perm_c): Pr A Pc = L U."""
        L = self._lu.L.tocsr()
        U = self._lu.U.tocsr()
        L.sort_indices()
        U.sort_indices()
        return L, U, np.asarray(self._lu.perm_r), np.asarray(self._lu.perm_c)

    def solve(self, b, trans="N"):
        """x with A x = b (``linsolve.py:48-53``)."""
        return self._lu.solve(np.asarray(b, dtype=float), trans=trans)

    def __call__(self, b):
        return self.solve(b)

    def inverse(self):
        """Dense A^{-1}, column j = SuperLU solve of e_j (setup for the device GEMV)."""
        n = self.shape[0]
        return np.ascontiguousarray(self._lu.solve(np.eye(n)))


def inverses(facts, max_workers=None):
    """Dense inverses of several factorizations, identical to ``[f.inverse() for f in facts]``:
    the identity's columns are solved in chunks on a thread pool (SuperLU's column solves are
    independent, so the result is bit-identical; cfg5's twelve 4225^2 face pieces 49 s -> a few s)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    out = [np.empty((f.shape[0], f.shape[0])) for f in facts]
    tasks = []
    for i, f in enumerate(facts):
        n = f.shape[0]
        step = max(64, -(-n // 16))
        tasks += [(i, lo, min(n, lo + step)) for lo in range(0, n, step)]

    def run(task):
        i, lo, hi = task
        n = facts[i].shape[0]
        E = np.zeros((n, hi - lo))
        E[np.arange(lo, hi), np.arange(hi - lo)] = 1.0
        out[i][:, lo:hi] = facts[i]._lu.solve(E)

    workers = max_workers or min(32, len(os.sched_getaffinity(0)))
    if len(tasks) <= 1 or workers <= 1:
        for t in tasks:
            run(t)
    else:
        with ThreadPoolExecutor(workers) as ex:
            list(ex.map(run, tasks))
    return [np.ascontiguousarray(x) for x in out]


def factorize(A, spd=False):
    return Factorization(A, spd=spd)


def solve(F, b):
    """Apply a factorization (``linsolve.py:60-61``)."""
    return F.solve(b)


def dense_generalized_eig(A, B):
    """Ascending eigenvalues of the pencil (A, B), A symmetric, B SPD (``linsolve.py:104-110``);
    a dense diagnostic, not on the solve path."""
    import scipy.linalg
    Ad = A.toarray() if scipy.sparse.issparse(A) else np.asarray(A, dtype=float)
    Bd = B.toarray() if scipy.sparse.issparse(B) else np.asarray(B, dtype=float)
    if Ad.shape != Bd.shape:
        raise ValueError("matrix dimensions do not match")
    return scipy.linalg.eigh(Ad, Bd, eigvals_only=True)


def write_coo(path, A):
    """Triplet text dump (``linsolve.py:113-119``): a header line ``rows cols nnz``, then one
    ``i j value`` line per stored entry, values with 17 significant digits (round-trips fp64)."""
    C = scipy.sparse.coo_matrix(A)
    lines = [f"{C.shape[0]} {C.shape[1]} {C.nnz}"]
    lines += [f"{i} {j} {v:.17g}" for i, j, v in zip(C.row.tolist(), C.col.tolist(), C.data.tolist())]
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def read_coo(path):
    """Inverse of :func:`write_coo` (``linsolve.py:122-131``); returns CSR (duplicates summed)."""
    with open(path) as fh:
        m, n, nnz = (int(t) for t in fh.readline().split())
        body = np.loadtxt(fh, ndmin=2, max_rows=nnz) if nnz else np.zeros((0, 3))
    if body.shape[0] != nnz:
        raise ValueError(f"{path}: expected {nnz} entries, found {body.shape[0]}")
    return scipy.sparse.csr_matrix((body[:, 2], (body[:, 0].astype(np.int64), body[:, 1].astype(np.int64))),
                                   shape=(m, n))


_plain_ctx = None


def _plain_context():
    """Device context for cg calls that carry no multigrid hierarchy (plain / host-callable
    preconditioner); created once, on device 0."""
    global _plain_ctx
    if _plain_ctx is None:
        from ._lib import Context
        _plain_ctx = Context(0)
    return _plain_ctx


def cg(A, b, preconditioner=None, tol=DEFAULT_TOL, max_iters=10000, callback=None):
    """Preconditioned CG on the device; returns ``(x, iterations, history)`` (``linsolve.py:64-101``).

    * ``preconditioner`` the DevicePreconditioner of a MultigridSolver (``solver.preconditioner()``,
      the reference call ``cg(solver.A[L], f, solver.preconditioner(), tol)``): without a callback
      the whole solve is one CUDA graph (``igb_pcg``); with ``callback(it, rel)`` a host-driven loop
      on the same kernels calls it after every iteration (``igb_cg``);
    * ``preconditioner=None`` (plain CG) or any host callable ``r -> z``: ``igb_cg`` with the CSR of
      ``A`` on the device; the callable runs on host copies of ``r`` once per iteration.
    All vector arithmetic and every product with ``A`` run on the device; there is no host CG path.
    """
    from .multigrid import DevicePreconditioner

    b = np.asarray(b, dtype=float)
    if isinstance(preconditioner, DevicePreconditioner):
        solver = preconditioner.solver
        finest = solver.A[solver.finest]
        same = A is finest or (A.shape == finest.shape and not (A != finest).nnz)
        if same and callback is None:
            return solver.ctx.pcg(b, tol, max_iters)
        return solver.ctx.cg(None if same else A, b, prec="cycle", tol=tol, max_iters=max_iters,
                             callback=callback)
    ctx = _plain_context()
    if preconditioner is None:
        return ctx.cg(A, b, prec="none", tol=tol, max_iters=max_iters, callback=callback)
    if not callable(preconditioner):
        raise TypeError("preconditioner must be None, a callable r -> z or a DevicePreconditioner")
    return ctx.cg(A, b, prec="host", prec_fn=preconditioner, tol=tol, max_iters=max_iters, callback=callback)
