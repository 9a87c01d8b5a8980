"""Univariate B-spline spaces on [0, 1] (host-side setup).

Same public surface as the reference's ``igamg.bspline`` (``bspline.py:15-27``):
open uniform knot vectors, Cox-de Boor evaluation with derivatives, Greville
abscissae, Gauss rules, 1-D mass/stiffness Gram matrices, dyadic two-scale
refinement and the reduced split used by the subspace-corrected mass smoother.

Everything here is host setup; nothing runs on the device.  The difference
from the reference is the evaluation layout: basis tables are computed for a
whole batch of points at once (arrays of shape ``(npts, p+1)``) instead of a
Python loop over points, which is what makes large-level assembly cheap.
The per-point arithmetic is the textbook recurrence (Piegl & Tiller A2.2 /
A2.3), so values agree with the reference to the last bit in practice.
"""

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse

__all__ = [
    "UnivariateSplineSpace",
    "ReducedSplit",
    "open_knot_vector",
    "eval_basis",
    "eval_basis_batch",
    "basis_matrices",
    "greville_points",
    "univariate_mass",
    "univariate_stiffness",
    "two_scale_refine",
    "reduced_split",
    "gauss_points",
    "interior_matrix",
]


@dataclass(frozen=True)
class UnivariateSplineSpace:
    """Degree-``p`` spline space on an open knot vector over [0, 1].

    Mirrors ``bspline.py:30-93`` (validation, ``n``, breakpoints, meshsize,
    value equality and hashing on (degree, knots)).
    """

    degree: int
    knots: np.ndarray = field(repr=False)

    def __post_init__(self):
        p = int(self.degree)
        kv = np.asarray(self.knots, dtype=float)
        if p < 1:
            raise ValueError("spline degree must be >= 1")
        if np.any(np.diff(kv) < 0):
            raise ValueError("knot vector must be non-decreasing")
        head, tail = kv[: p + 1], kv[-(p + 1):]
        if not (np.all(head == kv[0]) and kv[p + 1] > kv[0]):
            raise ValueError("first knot must have multiplicity exactly p+1")
        if not (np.all(tail == kv[-1]) and kv[-(p + 2)] < kv[-1]):
            raise ValueError("last knot must have multiplicity exactly p+1")
        object.__setattr__(self, "knots", kv)

    @property
    def n(self):
        return len(self.knots) - self.degree - 1

    @property
    def breakpoints(self):
        return np.unique(self.knots)

    @property
    def num_elements(self):
        return len(self.breakpoints) - 1

    @property
    def meshsize(self):
        return np.max(np.diff(self.breakpoints))

    def __eq__(self, other):
        if not isinstance(other, UnivariateSplineSpace):
            return NotImplemented
        return self.degree == other.degree and np.array_equal(self.knots, other.knots)

    def __hash__(self):
        return hash((self.degree, self.knots.tobytes()))


def open_knot_vector(p, coarse_elements, level=0):
    """Uniform open knot vector with ``coarse_elements * 2**level`` elements."""
    if p < 1:
        raise ValueError("degree must be >= 1")
    if coarse_elements < 1:
        raise ValueError("need at least one element")
    if level < 0:
        raise ValueError("level must be >= 0")
    ne = coarse_elements * 2 ** level
    knots = np.concatenate([np.zeros(p + 1), np.arange(1, ne) / ne, np.ones(p + 1)])
    return UnivariateSplineSpace(p, knots)


def _spans(space, x):
    """Knot-span index per point, last element closed on the right."""
    kv, n = space.knots, space.n
    idx = np.searchsorted(kv, x, side="right") - 1
    return np.where(x >= kv[n], n - 1, idx)


def eval_basis_batch(space, x, max_deriv=0):
    """Active basis functions (and derivatives) at many points.

    Returns ``(first, ders)`` with ``first`` int64 of shape ``(npts,)`` (index
    of the first active function) and ``ders`` of shape
    ``(max_deriv+1, npts, p+1)``.  Vectorised form of ``bspline.py:100-155``.
    """
    x = np.atleast_1d(np.asarray(x, dtype=float))
    if x.size and (x.min() < 0.0 or x.max() > 1.0):
        raise ValueError("evaluation point outside [0,1]")
    p, kv = space.degree, space.knots
    nq = x.shape[0]
    span = _spans(space, x)
    nd = min(max_deriv, p)

    # ndu[:, j, r]: upper triangle = basis values of degree j, lower = knot diffs
    ndu = np.zeros((nq, p + 1, p + 1))
    left = np.zeros((nq, p + 1))
    right = np.zeros((nq, p + 1))
    ndu[:, 0, 0] = 1.0
    for j in range(1, p + 1):
        left[:, j] = x - kv[span + 1 - j]
        right[:, j] = kv[span + j] - x
        saved = np.zeros(nq)
        for r in range(j):
            ndu[:, j, r] = right[:, r + 1] + left[:, j - r]
            temp = ndu[:, r, j - 1] / ndu[:, j, r]
            ndu[:, r, j] = saved + right[:, r + 1] * temp
            saved = left[:, j - r] * temp
        ndu[:, j, j] = saved

    ders = np.zeros((max_deriv + 1, nq, p + 1))
    ders[0] = ndu[:, :, p]
    if nd > 0:
        a = np.zeros((2, nq, p + 1))
        for r in range(p + 1):
            s1, s2 = 0, 1
            a[0, :, 0] = 1.0
            for k in range(1, nd + 1):
                d = np.zeros(nq)
                rk, pk = r - k, p - k
                if r >= k:
                    a[s2, :, 0] = a[s1, :, 0] / ndu[:, pk + 1, rk]
                    d = a[s2, :, 0] * ndu[:, rk, pk]
                j1 = 1 if rk >= -1 else -rk
                j2 = k - 1 if r - 1 <= pk else p - r
                for j in range(j1, j2 + 1):
                    a[s2, :, j] = (a[s1, :, j] - a[s1, :, j - 1]) / ndu[:, pk + 1, rk + j]
                    d = d + a[s2, :, j] * ndu[:, rk + j, pk]
                if r <= pk:
                    a[s2, :, k] = -a[s1, :, k - 1] / ndu[:, pk + 1, r]
                    d = d + a[s2, :, k] * ndu[:, r, pk]
                ders[k, :, r] = d
                s1, s2 = s2, s1
        fact = p
        for k in range(1, nd + 1):
            ders[k] *= fact
            fact *= p - k
    return span - p, ders


def eval_basis(space, x, max_deriv=0):
    """Single-point form: ``(first_active_index, ders[(max_deriv+1), p+1])``."""
    if x < 0.0 or x > 1.0:
        raise ValueError(f"evaluation point {x} outside [0,1]")
    first, ders = eval_basis_batch(space, np.array([x], dtype=float), max_deriv)
    return int(first[0]), ders[:, 0, :]


def basis_matrices(space, points, max_deriv=0):
    """Sparse collocation matrices ``[B0, B1, ...]`` of shape (npts, n)."""
    pts = np.atleast_1d(np.asarray(points, dtype=float))
    p, n = space.degree, space.n
    first, ders = eval_basis_batch(space, pts, max_deriv)
    nq = len(pts)
    rows = np.repeat(np.arange(nq), p + 1)
    cols = (first[:, None] + np.arange(p + 1)[None, :]).ravel()
    return [
        scipy.sparse.csr_matrix((ders[k].ravel(), (rows, cols)), shape=(nq, n))
        for k in range(max_deriv + 1)
    ]


def greville_points(space):
    p, kv = space.degree, space.knots
    idx = np.arange(space.n)[:, None] + 1 + np.arange(p)[None, :]
    return kv[idx].mean(axis=1)


def gauss_points(space, npts=None):
    """Gauss-Legendre nodes/weights on every element (default p+1 per element)."""
    if npts is None:
        npts = space.degree + 1
    xg, wg = np.polynomial.legendre.leggauss(npts)
    brk = space.breakpoints
    a, b = brk[:-1], brk[1:]
    nodes = (0.5 * (b - a)[:, None] * (xg + 1.0)[None, :] + a[:, None]).ravel()
    weights = (0.5 * (b - a)[:, None] * wg[None, :]).ravel()
    return nodes, weights


def _gram(space, du, dv):
    """Banded Gram matrix sum_q w_q B_du[q,i] B_dv[q,j], accumulated in q order."""
    x, w = gauss_points(space)
    p, n = space.degree, space.n
    first, ders = eval_basis_batch(space, x, max(du, dv))
    left = ders[du] * w[:, None]  # (nq, p+1)
    right = ders[dv]
    # entry (first+a, first+b) += left[q,a] * right[q,b]; accumulate in q order
    vals = (left[:, :, None] * right[:, None, :]).reshape(len(x), -1)
    rows = np.repeat(first[:, None] + np.arange(p + 1)[None, :], p + 1, axis=1)
    cols = np.tile(first[:, None] + np.arange(p + 1)[None, :], (1, p + 1))
    dense = np.zeros((n, n))
    np.add.at(dense, (rows.ravel(), cols.ravel()), vals.ravel())
    return dense


def _symmetrized_csr(dense):
    G = scipy.sparse.csr_matrix(dense)
    return ((G + G.T) * 0.5).tocsr()


def univariate_mass(space):
    """n-by-n Gram matrix of the basis in L2(0,1) (``bspline.py:204-207``)."""
    return _symmetrized_csr(_gram(space, 0, 0))


def univariate_stiffness(space):
    """n-by-n Gram matrix of the derivatives (``bspline.py:210-213``)."""
    return _symmetrized_csr(_gram(space, 1, 1))


def two_scale_refine(space):
    """Insert every element midpoint; returns ``(fine_space, P)`` with P (n_f x n_c).

    Restates Boehm single-knot insertion (``bspline.py:216-246``) on a dense
    coefficient block: each insertion maps rows c -> alpha_i c_i + (1-alpha_i) c_{i-1}.
    """
    p = space.degree
    knots = space.knots.copy()
    brk = space.breakpoints
    C = np.eye(space.n)
    for t in 0.5 * (brk[:-1] + brk[1:]):
        n = len(knots) - p - 1
        k = int(np.searchsorted(knots, t, side="right")) - 1
        new = np.empty((n + 1, C.shape[1]))
        lo = max(k - p + 1, 0)
        new[:lo] = C[:lo]
        for i in range(lo, k + 1):
            alpha = (t - knots[i]) / (knots[i + p] - knots[i])
            new[i] = (1.0 - alpha) * C[i - 1] + alpha * C[i]
        new[k + 1:] = C[k:]
        C = new
        knots = np.insert(knots, k + 1, t)
    return UnivariateSplineSpace(p, knots), scipy.sparse.csr_matrix(C)


@dataclass(frozen=True)
class ReducedSplit:
    """Interior space = large subspace (+) mass-orthogonal complement (``bspline.py:249-269``)."""

    n_constraints: int
    large: np.ndarray = field(repr=False)
    complement: np.ndarray = field(repr=False)

    @property
    def n_large(self):
        return self.large.shape[1]

    @property
    def n_comp(self):
        return self.complement.shape[1]


def interior_matrix(mat):
    """Principal submatrix without the first and last row/column."""
    return mat[1:-1, 1:-1]


def reduced_split(space):
    """Large subspace = kernel of even-order endpoint derivative constraints.

    Follows ``bspline.py:277-318``: constraints of orders 2, 4, ..., 2*floor((p-1)/2)
    at both endpoints (h-normalised), kernel via SVD, complement = M^{-1} C^T,
    M-orthonormalised by a Cholesky factor.
    """
    p, n = space.degree, space.n
    n_int = n - 2
    if n_int < 1:
        raise ValueError("space has no interior basis functions")
    m = (p - 1) // 2
    orders = [2 * (j + 1) for j in range(m)]
    n_con = 2 * m
    if n_int < n_con:
        raise ValueError(
            f"interior space of dimension {n_int} cannot carry {n_con} constraints"
        )
    if n_con == 0:
        return ReducedSplit(0, np.eye(n_int), np.zeros((n_int, 0)))
    C = np.zeros((n_con, n_int))
    h = space.meshsize
    for side, x in enumerate((0.0, 1.0)):
        first, ders = eval_basis(space, x, max(orders))
        for r, order in enumerate(orders):
            row = ders[order] * h ** order
            for j in range(p + 1):
                col = first + j - 1
                if 0 <= col < n_int:
                    C[side * m + r, col] += row[j]
    _, sv, Vt = np.linalg.svd(C)
    rank = int(np.sum(sv > max(C.shape) * np.finfo(float).eps * sv[0]))
    large = Vt[rank:].T
    M_int = interior_matrix(univariate_mass(space).toarray())
    comp = np.linalg.solve(M_int, C.T)
    G = comp.T @ M_int @ comp
    comp = comp @ np.linalg.inv(np.linalg.cholesky(G)).T
    return ReducedSplit(n_con, large, comp)
