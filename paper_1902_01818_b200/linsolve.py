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

__all__ = ["Factorization", "factorize", "cg", "DEFAULT_TOL"]

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

    def inverse(self):
        """Dense A^{-1}, column j = SuperLU solve of e_j (setup for the device GEMV)."""
        n = self.shape[0]
        return np.ascontiguousarray(self._lu.solve(np.eye(n)))


def factorize(A, spd=False):
    return Factorization(A, spd=spd)


def cg(A, b, preconditioner=None, tol=DEFAULT_TOL, max_iters=10000, callback=None):
    """Preconditioned CG on the device; returns ``(x, iterations, history)``.

    ``preconditioner`` must be the device preconditioner of a MultigridSolver
    whose finest operator is ``A`` (the reference call
    ``cg(solver.A[L], f, solver.preconditioner(), tol)``).  ``callback(it, rel)``
    is invoked after the solve for every history entry.
    """
    from .multigrid import DevicePreconditioner

    if not isinstance(preconditioner, DevicePreconditioner):
        raise TypeError(
            "device cg needs the DevicePreconditioner of a MultigridSolver "
            "(solver.preconditioner()); there is no host CG path")
    solver = preconditioner.solver
    if A is not solver.A[solver.finest] and (A.shape != solver.A[solver.finest].shape or
                                             (A != solver.A[solver.finest]).nnz):
        raise ValueError("cg operator differs from the preconditioner's finest matrix")
    b = np.asarray(b, dtype=float)
    x, its, history = solver.ctx.pcg(b, tol, max_iters)
    if callback is not None:
        for it, rel in enumerate(history, start=1):
            callback(it, rel)
    return x, its, history
