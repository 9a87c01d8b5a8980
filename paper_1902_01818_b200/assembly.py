"""Discrete hierarchies and assembly (host-side setup).

Public surface of the reference's ``igamg.assembly`` (``assembly.py:24-35``):
``build_hierarchy``, ``DiscreteHierarchy``, ``LevelDofs``, ``assemble_level``,
``assemble_rhs``, ``prolongation``, ``ManufacturedProblem``,
``Assumption2Error``.  Setup stays on the host (as in the reference); this
module feeds the device solve with ``A_L``, ``P_l`` and ``f``.

Design differences from the reference (same results up to summation order):

* DoF classes come from one connected-components pass instead of a Python
  union-find; the class root is the smallest block index of the class, which
  is exactly what the reference's min-root union produces (``assembly.py:61-80``).
* Bulk matrices of non-affine patches use sum factorisation on a banded
  representation ``Kb[i0, o0, i1, o1]`` (entry (i0,i1) x (i0+o0, i1+o1)):
  quadrature is contracted one direction at a time, element block by element
  block, instead of forming Kronecker collocation matrices with ~(p+1)^d
  nonzeros per quadrature point (``assembly.py:346-365``).
* Reduction to free DoFs maps COO entries through ``free_of_block`` instead of
  the ``Z^T A Z`` triple product (``assembly.py:591-608``).
"""

import itertools
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse
import scipy.sparse.csgraph

from . import bspline as bs
from . import _setup_native
from . import geometry as geom

__all__ = [
    "Assumption2Error",
    "ManufacturedProblem",
    "SourceProblem",
    "LevelDofs",
    "DiscreteHierarchy",
    "AssembledLevel",
    "build_hierarchy",
    "build_dofs",
    "assemble_level",
    "assemble_rhs",
    "solution_coefficients",
    "l2_error",
    "matrix_free_data",
    "check_coercivity",
    "geometry_condition_diagnostic",
    "prolongation",
]


class Assumption2Error(ValueError):
    """Conforming coupling requested for non-matching interface spaces."""


@dataclass(frozen=True)
class ManufacturedProblem:
    """u = prod sin(pi x_a), f = d pi^2 u, g = u (``assembly.py:42-55``)."""

    dim: int

    def exact(self, X):
        return np.prod(np.sin(np.pi * np.asarray(X)), axis=-1)

    def source(self, X):
        return self.dim * np.pi ** 2 * self.exact(X)

    def dirichlet(self, X):
        return self.exact(X)


@dataclass(frozen=True)
class SourceProblem:
    """Arbitrary source ``f(X)`` with Dirichlet data ``g(X)`` (0 if None)."""

    f: object
    g: object = None

    def source(self, X):
        return np.asarray(self.f(np.asarray(X)), dtype=float) * np.ones(np.shape(X)[:-1])

    def dirichlet(self, X):
        if self.g is None:
            return np.zeros(np.shape(X)[:-1])
        return np.asarray(self.g(np.asarray(X)), dtype=float)


# -- degrees of freedom --------------------------------------------------------


@dataclass
class LevelDofs:
    """Numbering of one level (``assembly.py:83-135``), array form.

    ``class_of[b]`` is the smallest block index in b's class; ``free_of_block``
    and ``dir_of_block`` give the free / Dirichlet id of every block index
    (-1 where not applicable).  Free ids follow ascending class root.
    """

    dims: list
    offsets: np.ndarray
    class_of: np.ndarray
    free_of_block: np.ndarray
    dir_of_block: np.ndarray
    n_free: int
    n_dirichlet: int

    @property
    def n_block(self):
        return int(self.offsets[-1])

    @property
    def free_id(self):
        roots = np.flatnonzero((self.class_of == np.arange(self.n_block)) & (self.free_of_block >= 0))
        return dict(zip(roots.tolist(), self.free_of_block[roots].tolist()))

    @property
    def dirichlet_id(self):
        roots = np.flatnonzero((self.class_of == np.arange(self.n_block)) & (self.dir_of_block >= 0))
        return dict(zip(roots.tolist(), self.dir_of_block[roots].tolist()))

    def block_index(self, k, multi):
        return self.offsets[k] + np.ravel_multi_index(multi, self.dims[k])

    def free_of(self, k, multi):
        return int(self.free_of_block[self.block_index(k, multi)])

    def free_representatives(self):
        """Block index of the class root of every free DoF (free id order)."""
        rep = np.empty(self.n_free, dtype=np.int64)
        roots = np.flatnonzero((self.class_of == np.arange(self.n_block)) & (self.free_of_block >= 0))
        rep[self.free_of_block[roots]] = roots
        return rep

    def patch_of_block(self, b):
        return np.searchsorted(self.offsets, b, side="right") - 1

    def scatter_matrices(self):
        n = self.n_block
        f = self.free_of_block
        dmask = self.dir_of_block >= 0
        rows = np.arange(n)
        Zf = scipy.sparse.csr_matrix(
            (np.ones(int((f >= 0).sum())), (rows[f >= 0], f[f >= 0])), shape=(n, self.n_free))
        Zd = scipy.sparse.csr_matrix(
            (np.ones(int(dmask.sum())), (rows[dmask], self.dir_of_block[dmask])),
            shape=(n, self.n_dirichlet))
        return Zf, Zd


def _side_lattice(dims, side):
    """Multi-index arrays of the DoF layer on ``side`` (C order over tangential axes)."""
    d = len(dims)
    tang = side.tangential_axes(d)
    sizes = [dims[a] for a in tang]
    grids = np.meshgrid(*[np.arange(s) for s in sizes], indexing="ij")
    multi = []
    for a in range(d):
        if a == side.axis:
            multi.append(np.full(grids[0].shape, side.end * (dims[a] - 1)))
        else:
            multi.append(grids[tang.index(a)])
    return multi, sizes


def _check_assumption2(per_patch, iface, d):
    tk = iface.side_k.tangential_axes(d)
    tl = iface.side_l.tangential_axes(d)
    for i in range(d - 1):
        sk = per_patch[iface.k][tk[i]]
        sl = per_patch[iface.l][tl[iface.orientation.perm[i]]]
        same = sk.degree == sl.degree and len(sk.knots) == len(sl.knots)
        if same:
            kl = sl.knots if not iface.orientation.flips[i] else 1.0 - sl.knots[::-1]
            same = np.allclose(sk.knots, kl, atol=1e-12)
        if not same:
            raise Assumption2Error(
                f"interface between patches {iface.k} and {iface.l}: tangential "
                "spaces do not match (degree/knot vector differ)")


def _interface_block_pairs(dims, offsets, iface, d):
    """Block indices of matched DoFs on the two sides of a conforming interface."""
    multi_k, sizes = _side_lattice(dims[iface.k], iface.side_k)
    grids = np.meshgrid(*[np.arange(s) for s in sizes], indexing="ij")
    tl = iface.side_l.tangential_axes(d)
    along_l = {}
    for i in range(d - 1):
        ax_l = tl[iface.orientation.perm[i]]
        n_t = dims[iface.l][ax_l]
        along_l[ax_l] = (n_t - 1 - grids[i]) if iface.orientation.flips[i] else grids[i]
    multi_l = []
    for a in range(d):
        if a == iface.side_l.axis:
            multi_l.append(np.full(grids[0].shape, iface.side_l.end * (dims[iface.l][a] - 1)))
        else:
            multi_l.append(along_l[a])
    bk = offsets[iface.k] + np.ravel_multi_index([m.ravel() for m in multi_k], dims[iface.k])
    bl = offsets[iface.l] + np.ravel_multi_index([m.ravel() for m in multi_l], dims[iface.l])
    return bk, bl


def build_dofs(domain, per_patch, mode):
    """Global numbering of one level (``assembly.py:236-292`` semantics)."""
    d = domain.dim
    dims = [tuple(s.n for s in spaces) for spaces in per_patch]
    sizes = [int(np.prod(dd)) for dd in dims]
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n_block = int(offsets[-1])

    if mode == "conforming" and domain.interfaces:
        pairs = []
        for iface in domain.interfaces:
            _check_assumption2(per_patch, iface, d)
            pairs.append(_interface_block_pairs(dims, offsets, iface, d))
        a = np.concatenate([p[0] for p in pairs])
        b = np.concatenate([p[1] for p in pairs])
        g = scipy.sparse.coo_matrix((np.ones(len(a)), (a, b)), shape=(n_block, n_block))
        _, label = scipy.sparse.csgraph.connected_components(g, directed=False)
        root_of_label = np.full(label.max() + 1, n_block, dtype=np.int64)
        np.minimum.at(root_of_label, label, np.arange(n_block))
        class_of = root_of_label[label]
    else:
        class_of = np.arange(n_block, dtype=np.int64)

    is_dir_root = np.zeros(n_block, dtype=bool)
    for k, side in domain.boundary:
        multi, _ = _side_lattice(dims[k], side)
        blk = offsets[k] + np.ravel_multi_index([m.ravel() for m in multi], dims[k])
        is_dir_root[class_of[blk]] = True
    is_root = class_of == np.arange(n_block)
    free_root = is_root & ~is_dir_root
    dir_root = is_root & is_dir_root
    root_free = np.cumsum(free_root) - 1
    root_dir = np.cumsum(dir_root) - 1
    free_of_block = np.where(free_root[class_of], root_free[class_of], -1).astype(np.int64)
    dir_of_block = np.where(dir_root[class_of], root_dir[class_of], -1).astype(np.int64)
    return LevelDofs(dims, offsets, class_of, free_of_block, dir_of_block,
                     int(free_root.sum()), int(dir_root.sum()))


# -- hierarchy ----------------------------------------------------------------


@dataclass
class DiscreteHierarchy:
    """Per-level, per-patch tensor spaces plus numberings (``assembly.py:153-180``)."""

    domain: geom.MultiPatchDomain
    p: int
    L: int
    mode: str
    space_rule: str
    coarse_elements: int = 1
    spaces: list = field(default_factory=list)
    dofs: list = field(default_factory=list)

    @property
    def dim(self):
        return self.domain.dim

    def n_free(self, level):
        return self.dofs[level].n_free

    def finest_meshsize(self):
        return min(s.meshsize for patch in self.spaces[self.L] for s in patch)

    def patch_meshsize(self, level, k):
        return max(s.meshsize for s in self.spaces[level][k])


def _patch_space(p, rule, k, level, coarse_elements):
    if rule == "matching":
        deg, lev = p, level
    elif rule == "nonmatching":
        r = k % 3
        deg = p + 1 if r == 1 else p
        lev = level if r == 0 else max(level - 1, 0)
    else:
        raise ValueError(f"unknown space rule {rule!r}")
    return bs.open_knot_vector(deg, coarse_elements, lev)


def build_hierarchy(domain, p, L, mode="conforming", space_rule="matching", coarse_elements=1):
    """Spaces and numberings for levels 0..L (``assembly.py:195-215``)."""
    if mode not in ("conforming", "dg"):
        raise ValueError(f"unknown coupling mode {mode!r}")
    if mode == "conforming" and space_rule != "matching":
        raise Assumption2Error("conforming coupling requires matching spaces on the interfaces")
    if L < 1:
        raise ValueError("need at least one refinement level")
    hier = DiscreteHierarchy(domain, p, L, mode, space_rule, coarse_elements)
    for level in range(L + 1):
        per_patch = []
        for k in range(domain.num_patches):
            s = _patch_space(p, space_rule, k, level, coarse_elements)
            per_patch.append(tuple(s for _ in range(domain.dim)))
        hier.spaces.append(per_patch)
        hier.dofs.append(build_dofs(domain, per_patch, mode))
    return hier


def hierarchy_from_spaces(domain, p, L, mode, spaces_per_level, space_rule="custom"):
    """Hierarchy with caller-given per-level, per-patch spaces (e.g. config 3's 64/128/256 grids)."""
    hier = DiscreteHierarchy(domain, p, L, mode, space_rule)
    for level in range(L + 1):
        per_patch = [tuple(s) for s in spaces_per_level[level]]
        hier.spaces.append(per_patch)
        hier.dofs.append(build_dofs(domain, per_patch, mode))
    return hier


# -- bulk matrices ---------------------------------------------------------------


def _probe_jacobian(patch):
    """Constant diagonal Jacobian (scale factors) or None (``assembly.py:317-327``)."""
    _, J = patch.eval_grid([np.array([0.0, 0.37, 1.0])] * patch.dim)
    J = J.reshape(-1, patch.dim, patch.dim)
    if np.abs(J - J[0]).max() > 1e-13:
        return None
    J0 = J[0]
    if np.abs(J0 - np.diag(np.diag(J0))).max() > 1e-13:
        return None
    return np.diag(J0).copy()


def _kron_chain(mats):
    out = mats[0]
    for m in mats[1:]:
        out = scipy.sparse.kron(out, m, format="csr")
    return out


def _element_tables(space):
    """Quadrature per element: nodes, weights, values/derivs (nel, nqe, p+1), first index."""
    x, w = bs.gauss_points(space)
    first, ders = bs.eval_basis_batch(space, x, 1)
    nel = space.num_elements
    nqe = len(x) // nel
    p = space.degree
    return (x, w, ders[0].reshape(nel, nqe, p + 1), ders[1].reshape(nel, nqe, p + 1),
            first.reshape(nel, nqe)[:, 0])


def _pair_tables(U, V):
    """E[e, q, a*(p+1)+b] = U[e,q,a] * V[e,q,b]."""
    nel, nqe, m = U.shape
    return (U[:, :, :, None] * V[:, :, None, :]).reshape(nel, nqe, m * m)


def _band_2d(C, tab0, tab1, U0, V0, U1, V1, p0, p1, n0, n1):
    """Kb[i0, o0+p0, i1, o1+p1] = sum_{q0,q1} U0[q0,i0]V0[q0,i0+o0] C[q0,q1] U1[q1,i1]V1[q1,i1+o1]."""
    nel0, nqe0, first0 = tab0
    nel1, nqe1, first1 = tab1
    w0, w1 = 2 * p0 + 1, 2 * p1 + 1
    E0 = _pair_tables(U0, V0)  # (nel0, nqe0, (p0+1)^2)
    E1 = _pair_tables(U1, V1)
    nq0 = C.shape[0]
    # step 1: Z[q0, i1, o1] = sum_q1 C[q0,q1] E1[q1, (i1,o1)]
    Cr = C.reshape(nq0, nel1, nqe1)
    contrib = np.einsum("xeq,eqk->xek", Cr, E1, optimize=True)  # (nq0, nel1, (p1+1)^2)
    Z = np.zeros((nq0, n1, w1))
    for a in range(p1 + 1):
        for b in range(p1 + 1):
            Z[:, first1 + a, b - a + p1] += contrib[:, :, a * (p1 + 1) + b]
    # step 2: Kb[i0, o0, :, :] += E0[q0,(i0,o0)] Z[q0, :, :] per element, in chunks
    Kb = np.zeros((n0, w0, n1 * w1))
    Zr = Z.reshape(nel0, nqe0, n1 * w1)
    chunk = max(1, int(2e8 // max(1, (p0 + 1) ** 2 * n1 * w1)))
    for e_lo in range(0, nel0, chunk):
        e_hi = min(nel0, e_lo + chunk)
        part = np.matmul(np.swapaxes(E0[e_lo:e_hi], 1, 2), Zr[e_lo:e_hi])  # (ne, (p0+1)^2, n1*w1)
        for a in range(p0 + 1):
            for b in range(p0 + 1):
                Kb[first0[e_lo:e_hi] + a, b - a + p0, :] += part[:, a * (p0 + 1) + b, :]
    return Kb.reshape(n0, w0, n1, w1)


def _band_transpose(Kb, p0, p1):
    """Band form of the transposed operator: KbT[i0,o0,i1,o1] = Kb[i0+o0,-o0,i1+o1,-o1]."""
    n0, w0, n1, w1 = Kb.shape
    out = np.zeros_like(Kb)
    for o0 in range(-p0, p0 + 1):
        s0 = slice(max(0, -o0), min(n0, n0 - o0))
        t0 = slice(max(0, o0), min(n0, n0 + o0))
        for o1 in range(-p1, p1 + 1):
            s1 = slice(max(0, -o1), min(n1, n1 - o1))
            t1 = slice(max(0, o1), min(n1, n1 + o1))
            out[s0, o0 + p0, s1, o1 + p1] = Kb[t0, -o0 + p0, t1, -o1 + p1]
    return out


def _band_to_csr(Kb, p0, p1):
    """Banded 2-D operator -> CSR in lexicographic (i0 slowest) numbering, sorted columns."""
    n0, w0, n1, w1 = Kb.shape
    i0 = np.arange(n0)[:, None, None, None]
    o0 = np.arange(-p0, p0 + 1)[None, :, None, None]
    i1 = np.arange(n1)[None, None, :, None]
    o1 = np.arange(-p1, p1 + 1)[None, None, None, :]
    j0, j1 = i0 + o0, i1 + o1
    valid = (j0 >= 0) & (j0 < n0) & (j1 >= 0) & (j1 < n1)
    valid = np.broadcast_to(valid, Kb.shape)
    cols = np.broadcast_to(j0 * n1 + j1, Kb.shape)
    # reorder to (i0, i1, o0, o1): rows major, columns ascending
    perm = (0, 2, 1, 3)
    v = valid.transpose(perm).reshape(n0 * n1, -1)
    data = Kb.transpose(perm).reshape(n0 * n1, -1)[v]
    idx = cols.transpose(perm).reshape(n0 * n1, -1)[v]
    indptr = np.concatenate([[0], np.cumsum(v.sum(axis=1))])
    return scipy.sparse.csr_matrix((data, idx, indptr), shape=(n0 * n1, n0 * n1))


def _bulk_matrices(patch, spaces, neglect_geometry=False, want_mass=True):
    """Per-patch stiffness (and mass) in the patch's tensor numbering (``assembly.py:330-365``)."""
    d = len(spaces)
    scal = np.ones(d) if neglect_geometry else _probe_jacobian(patch)
    if scal is not None:
        det = float(np.prod(scal))
        Ms = [bs.univariate_mass(s) for s in spaces]
        Ks = [bs.univariate_stiffness(s) for s in spaces]
        M = det * _kron_chain(Ms) if want_mass else None
        shape = (int(np.prod([s.n for s in spaces])),) * 2
        K = scipy.sparse.csr_matrix(shape)
        for a in range(d):
            K = K + (det / scal[a] ** 2) * _kron_chain([Ks[i] if i == a else Ms[i] for i in range(d)])
        return K.tocsr(), (M.tocsr() if M is not None else None)
    if d == 2:
        return _bulk_quadrature_2d(patch, spaces, want_mass)
    return _bulk_quadrature_generic(patch, spaces)


def _geometry_factors(patch, nodes, weights):
    _, J = patch.eval_grid(nodes)
    detJ = np.abs(np.linalg.det(J))
    if detJ.min() <= 0:
        raise geom.GeometryError("singular Jacobian at a quadrature point")
    Jinv = np.linalg.inv(J)
    G = np.einsum("...ac,...bc,...->...ab", Jinv, Jinv, detJ)
    wq = weights[0]
    for w in weights[1:]:
        wq = np.multiply.outer(wq, w)
    return wq, detJ, G


def _bulk_quadrature_2d(patch, spaces, want_mass):
    s0, s1 = spaces
    x0, w0, B0, D0, f0 = _element_tables(s0)
    x1, w1, B1, D1, f1 = _element_tables(s1)
    wq, detJ, G = _geometry_factors(patch, [x0, x1], [w0, w1])
    p0, p1, n0, n1 = s0.degree, s1.degree, s0.n, s1.n
    tab0 = (B0.shape[0], B0.shape[1], f0)
    tab1 = (B1.shape[0], B1.shape[1], f1)

    def band(C, U0, V0, U1, V1):
        return _band_2d(C, tab0, tab1, U0, V0, U1, V1, p0, p1, n0, n1)

    K00 = band(wq * G[..., 0, 0], D0, D0, B1, B1)
    K01 = band(wq * G[..., 0, 1], D0, B0, B1, D1)
    K11 = band(wq * G[..., 1, 1], B0, B0, D1, D1)
    Kb = ((K00 + K01) + _band_transpose(K01, p0, p1)) + K11
    K = _band_to_csr(Kb, p0, p1)
    M = _band_to_csr(band(wq * detJ, B0, B0, B1, B1), p0, p1) if want_mass else None
    return K, M


def _bulk_quadrature_generic(patch, spaces):
    """Reference-style collocation assembly for non-affine patches in d != 2."""
    d = len(spaces)
    nodes, weights, B, D = [], [], [], []
    for s in spaces:
        x, w = bs.gauss_points(s)
        b0, b1 = bs.basis_matrices(s, x, 1)
        nodes.append(x)
        weights.append(w)
        B.append(b0)
        D.append(b1)
    wq, detJ, G = _geometry_factors(patch, nodes, weights)
    Bk = [_kron_chain([D[i] if i == a else B[i] for i in range(d)]) for a in range(d)]
    B0 = _kron_chain(B)
    M = (B0.T @ scipy.sparse.diags((wq * detJ).ravel()) @ B0).tocsr()
    K = scipy.sparse.csr_matrix(M.shape)
    for a in range(d):
        for b in range(a, d):
            T = (Bk[a].T @ scipy.sparse.diags((wq * G[..., a, b]).ravel()) @ Bk[b]).tocsr()
            K = K + T if a == b else K + T + T.T
    return K.tocsr(), M


# -- SIPG interface forms ------------------------------------------------------------


def _merged_breakpoints(a, b):
    v = np.sort(np.concatenate([a, b]))
    return v[np.concatenate([[True], np.diff(v) > 1e-12])]


def _side_traces(spaces, side, tang_points):
    """Value rows T and parameter-gradient rows G_b of the tensor basis on a side."""
    d = len(spaces)
    tang = side.tangential_axes(d)
    vals, ders = [], []
    for a in range(d):
        pts = np.array([float(side.end)]) if a == side.axis else tang_points[tang.index(a)]
        b0, b1 = bs.basis_matrices(spaces[a], pts, 1)
        vals.append(b0)
        ders.append(b1)
    T = _kron_chain(vals)
    G = [_kron_chain([ders[i] if i == b else vals[i] for i in range(d)]) for b in range(d)]
    return T, G


def _orientation_row_perm(orient, sizes_k):
    m = len(sizes_k)
    sizes_l = [0] * m
    for i in range(m):
        sizes_l[orient.perm[i]] = sizes_k[i]
    grids = np.meshgrid(*[np.arange(s) for s in sizes_k], indexing="ij")
    idx_l = [None] * m
    for i in range(m):
        idx_l[orient.perm[i]] = grids[i]
    return np.ravel_multi_index([g.ravel() for g in idx_l], sizes_l)


def _interface_forms(hier, level, iface, neglect_geometry):
    """Jump/average rows and surface weights of one interface (``assembly.py:436-517``)."""
    d = hier.dim
    domain = hier.domain
    dofs = hier.dofs[level]
    sk, sl = hier.spaces[level][iface.k], hier.spaces[level][iface.l]
    tk, tl = iface.side_k.tangential_axes(d), iface.side_l.tangential_axes(d)
    p_max = max(max(s.degree for s in sk), max(s.degree for s in sl))
    xg, wg = np.polynomial.legendre.leggauss(p_max + 1)
    axes, weights = [], []
    for i in range(d - 1):
        brk_l = sl[tl[iface.orientation.perm[i]]].breakpoints
        if iface.orientation.flips[i]:
            brk_l = np.sort(1.0 - brk_l)
        brk = _merged_breakpoints(sk[tk[i]].breakpoints, brk_l)
        a, b = brk[:-1], brk[1:]
        axes.append((0.5 * (b - a)[:, None] * (xg + 1) + a[:, None]).ravel())
        weights.append((0.5 * (b - a)[:, None] * np.broadcast_to(wg, (len(a), len(wg)))).ravel())
    sizes = [len(a) for a in axes]
    nq = int(np.prod(sizes))

    Tk, Gk = _side_traces(sk, iface.side_k, axes)
    axes_l = [None] * (d - 1)
    for i in range(d - 1):
        j = iface.orientation.perm[i]
        axes_l[j] = 1.0 - axes[i] if iface.orientation.flips[i] else axes[i]
    Tl, Gl = _side_traces(sl, iface.side_l, axes_l)
    rp = _orientation_row_perm(iface.orientation, sizes) if d == 3 else None
    if rp is not None:
        Tl = Tl[rp]
        Gl = [g[rp] for g in Gl]

    def full_axes(side, tang_pts):
        tang = side.tangential_axes(d)
        return [np.array([float(side.end)]) if a == side.axis else tang_pts[tang.index(a)]
                for a in range(d)]

    if neglect_geometry:
        Jk = np.broadcast_to(np.eye(d), (nq, d, d))
        Jl = Jk
    else:
        _, Jk = domain.patches[iface.k].eval_grid(full_axes(iface.side_k, axes))
        Jk = Jk.reshape(nq, d, d)
        _, Jl = domain.patches[iface.l].eval_grid(full_axes(iface.side_l, axes_l))
        Jl = Jl.reshape(-1, d, d)
        if rp is not None:
            Jl = Jl[rp]

    tangents = [Jk[:, :, a] for a in tk]
    if d == 2:
        surf = np.linalg.norm(tangents[0], axis=1)
    else:
        surf = np.linalg.norm(np.cross(tangents[0], tangents[1]), axis=1)
    wq = weights[0]
    for w in weights[1:]:
        wq = np.multiply.outer(wq, w)
    wsurf = wq.ravel() * surf

    nhat = np.zeros(d)
    nhat[iface.side_k.axis] = 1.0 if iface.side_k.end == 1 else -1.0
    n_phys = np.einsum("qba,b->qa", np.linalg.inv(Jk), nhat)
    n_phys /= np.linalg.norm(n_phys, axis=1)[:, None]

    def normal_rows(G, J):
        coef = np.einsum("qab,qb->qa", np.linalg.inv(J), n_phys)
        rows = scipy.sparse.csr_matrix(G[0].shape)
        for b in range(d):
            rows = rows + scipy.sparse.diags(coef[:, b]) @ G[b]
        return rows

    Jmp = scipy.sparse.hstack([Tk, -Tl], format="csr")
    Avg = scipy.sparse.hstack([0.5 * normal_rows(Gk, Jk), 0.5 * normal_rows(Gl, Jl)], format="csr")
    cols = np.concatenate([
        dofs.offsets[iface.k] + np.arange(int(np.prod(dofs.dims[iface.k]))),
        dofs.offsets[iface.l] + np.arange(int(np.prod(dofs.dims[iface.l]))),
    ])
    return Jmp, Avg, wsurf, cols, p_max


# -- level assembly ----------------------------------------------------------------


@dataclass
class AssembledLevel:
    """Free-DoF operator of one level plus Dirichlet coupling (``assembly.py:520-547``)."""

    level: int
    A: scipy.sparse.csr_matrix
    sigma: float
    h_L: float
    couple: scipy.sparse.csr_matrix = None
    dirichlet_points: np.ndarray = None
    K: scipy.sparse.csr_matrix = None
    M: scipy.sparse.csr_matrix = None
    J: scipy.sparse.csr_matrix = None
    B: scipy.sparse.csr_matrix = None
    Q: scipy.sparse.csr_matrix = None

    @property
    def n(self):
        return self.A.shape[0]


def _map_coo(mat, row_map, col_map, row_off=0, col_off=0):
    coo = mat.tocoo()
    r = row_map[coo.row + row_off]
    c = col_map[coo.col + col_off]
    keep = (r >= 0) & (c >= 0)
    return r[keep], c[keep], coo.data[keep]


def _coo_sum(parts, shape):
    if not parts:
        return scipy.sparse.csr_matrix(shape)
    r = np.concatenate([p[0] for p in parts])
    c = np.concatenate([p[1] for p in parts])
    v = np.concatenate([p[2] for p in parts])
    idx_dtype = np.int32 if max(shape) < 2 ** 31 - 1 else np.int64
    out = scipy.sparse.coo_matrix((v, (r.astype(idx_dtype), c.astype(idx_dtype))), shape=shape).tocsr()
    out.sum_duplicates()
    out.sort_indices()
    return out


def assemble_level(hier, level, sigma=5.0, neglect_geometry=False, parts=("A",)):
    """Assemble the free-DoF operator of one level (``assembly.py:550-614``).

    ``A = K + (sigma/h_L) * sum_iface p_int^2 J_iface - B - B^T`` (dG) or ``A = K``
    (conforming), reduced to free DoFs, plus the free x Dirichlet coupling block
    used by ``assemble_rhs``.  ``parts`` may add "K", "M", "J", "B", "Q".
    """
    domain = hier.domain
    dofs = hier.dofs[level]
    n_block = dofs.n_block
    fob, dob = dofs.free_of_block, dofs.dir_of_block
    want = set(parts) | {"A"}
    want_mass = "M" in want
    if hier.mode == "conforming" and not (want - {"A", "K", "Q"}):
        native = _native_kron_level(hier, level, neglect_geometry)
        if native is not None:
            A, couple = native
            asm = AssembledLevel(level=level, A=A, sigma=sigma, h_L=hier.finest_meshsize(), couple=couple,
                                 dirichlet_points=_dirichlet_points(hier, level, neglect_geometry))
            if want & {"K", "Q"}:
                asm.K = asm.Q = A
            asym, amax = _setup_native.max_asym(A)
            if asym > 1e-10 * amax:
                raise AssertionError("assembled operator lost symmetry")
            return asm

    Kp, Mp = [], []
    for k in range(domain.num_patches):
        K, M = _bulk_matrices(domain.patches[k], hier.spaces[level][k], neglect_geometry, want_mass)
        Kp.append(K)
        Mp.append(M)

    h_L = hier.finest_meshsize()
    iface_blocks = []  # block-numbered interface matrices (dG)
    J_blk = Jpen_blk = B_blk = None
    if hier.mode == "dg" and domain.interfaces:
        J_blk = scipy.sparse.csr_matrix((n_block, n_block))
        Jpen_blk = scipy.sparse.csr_matrix((n_block, n_block))
        B_blk = scipy.sparse.csr_matrix((n_block, n_block))
        for iface in domain.interfaces:
            Jmp, Avg, wsurf, cols, p_int = _interface_forms(hier, level, iface, neglect_geometry)
            W = scipy.sparse.diags(wsurf)
            Jloc = (Jmp.T @ W @ Jmp).tocoo()
            Bloc = (Avg.T @ W @ Jmp).tocoo()
            Jg = scipy.sparse.csr_matrix((Jloc.data, (cols[Jloc.row], cols[Jloc.col])), shape=(n_block,) * 2)
            Bg = scipy.sparse.csr_matrix((Bloc.data, (cols[Bloc.row], cols[Bloc.col])), shape=(n_block,) * 2)
            J_blk = J_blk + Jg
            Jpen_blk = Jpen_blk + p_int ** 2 * Jg
            B_blk = B_blk + Bg
        iface_blocks = [(sigma / h_L) * Jpen_blk - B_blk - B_blk.T]

    def reduce_blockdiag(mats, row_map, col_map, extra=()):
        pieces = []
        for k, m in enumerate(mats):
            off = int(dofs.offsets[k])
            pieces.append(_map_coo(m, row_map, col_map, off, off))
        for m in extra:
            pieces.append(_map_coo(m, row_map, col_map))
        return pieces

    shape_ff = (dofs.n_free, dofs.n_free)
    A = _coo_sum(reduce_blockdiag(Kp, fob, fob, iface_blocks), shape_ff)
    couple = _coo_sum(reduce_blockdiag(Kp, fob, dob, iface_blocks), (dofs.n_free, dofs.n_dirichlet))

    asm = AssembledLevel(level=level, A=A, sigma=sigma, h_L=h_L, couple=couple,
                         dirichlet_points=_dirichlet_points(hier, level, neglect_geometry))
    if "K" in want or "Q" in want:
        asm.K = _coo_sum(reduce_blockdiag(Kp, fob, fob), shape_ff)
    if want_mass:
        asm.M = _coo_sum(reduce_blockdiag(Mp, fob, fob), shape_ff)
    if J_blk is not None:
        if "J" in want:
            asm.J = _coo_sum([_map_coo(J_blk, fob, fob)], shape_ff)
        if "B" in want:
            asm.B = _coo_sum([_map_coo(B_blk, fob, fob)], shape_ff)
        if "Q" in want:
            asm.Q = _coo_sum(reduce_blockdiag(Kp, fob, fob, [(sigma / h_L) * Jpen_blk]), shape_ff)
    elif "Q" in want:
        asm.Q = asm.K
    asym = abs(A - A.T)
    if asym.nnz and asym.max() > 1e-10 * abs(A).max():
        raise AssertionError("assembled operator lost symmetry")
    return asm


def _native_kron_level(hier, level, neglect_geometry):
    """(A, couple) of a conforming level whose patches all take the Kronecker branch of
    ``_bulk_matrices`` (constant diagonal Jacobian, ``assembly.py:333-344``), assembled and reduced
    to free DoFs natively (csrc/host_setup.cpp), bit-identical to ``_coo_sum(reduce_blockdiag(...))``
    of the SciPy path; None when the library is unavailable or a patch is not affine."""
    if _setup_native.lib() is None:
        return None
    dofs = hier.dofs[level]
    d = hier.dim
    coef, oned, dims = [], [], []
    for k in range(hier.domain.num_patches):
        scal = np.ones(d) if neglect_geometry else _probe_jacobian(hier.domain.patches[k])
        if scal is None:
            return None
        det = float(np.prod(scal))
        coef.append([det / scal[a] ** 2 for a in range(d)])
        per = []
        for s in hier.spaces[level][k]:
            M = bs.univariate_mass(s).tocsr()
            K = bs.univariate_stiffness(s).tocsr()
            if not (M.has_sorted_indices and K.has_sorted_indices and np.array_equal(M.indptr, K.indptr)
                    and np.array_equal(M.indices, K.indices)):
                return None
            per.append((M, K))
        oned.append(per)
        dims.append([s.n for s in hier.spaces[level][k]])
    bo = np.asarray(dofs.offsets, dtype=np.int64)
    A = _setup_native.kron_reduce(dims, coef, oned, bo, dofs.free_of_block, dofs.free_of_block,
                                  dofs.n_free, dofs.n_free)
    couple = _setup_native.kron_reduce(dims, coef, oned, bo, dofs.free_of_block, dofs.dir_of_block,
                                       dofs.n_free, dofs.n_dirichlet)
    return A, couple


def _dirichlet_points(hier, level, neglect_geometry):
    """Physical Greville point of each Dirichlet class (first member in block order)."""
    dofs = hier.dofs[level]
    pts = np.zeros((dofs.n_dirichlet, hier.dim))
    if dofs.n_dirichlet == 0:
        return pts
    done = np.zeros(dofs.n_dirichlet, dtype=bool)
    for k in range(hier.domain.num_patches):
        grev = [bs.greville_points(s) for s in hier.spaces[level][k]]
        if neglect_geometry:
            X = np.stack(np.meshgrid(*grev, indexing="ij"), axis=-1)
        else:
            X, _ = hier.domain.patches[k].eval_grid(grev)
        flat = X.reshape(-1, hier.dim)
        did = dofs.dir_of_block[dofs.offsets[k]:dofs.offsets[k + 1]]
        sel = np.flatnonzero(did >= 0)
        ids = did[sel]
        # first occurrence within this patch, and not already set by an earlier patch
        uniq, first = np.unique(ids, return_index=True)
        new = ~done[uniq]
        pts[uniq[new]] = flat[sel[first[new]]]
        done[uniq[new]] = True
    return pts


def _tensor_load(spaces, patch, problem):
    """Sum-factorised load vector B^T (w detJ f) of one patch (patch numbering)."""
    d = len(spaces)
    nodes, weights, Bd = [], [], []
    for s in spaces:
        x, w = bs.gauss_points(s)
        nodes.append(x)
        weights.append(w)
        Bd.append(bs.basis_matrices(s, x, 0)[0])
    scal = _probe_jacobian(patch)
    if scal is not None:
        # constant diagonal Jacobian (the Kronecker case of assembly.py:333-344): x_a depends on xi_a
        # only and det J is constant -- evaluate the map along each axis instead of on the full
        # quadrature grid (equal to rounding; 8 x 16.7M points on cfg5)
        X = np.empty(tuple(len(x) for x in nodes) + (d,))
        for a in range(d):
            Xa, _ = patch.eval_grid([nodes[b] if b == a else nodes[b][:1] for b in range(d)])
            shape = [1] * d
            shape[a] = -1
            X[..., a] = Xa[..., a].reshape(shape)
        detJ = abs(float(np.prod(scal)))
    else:
        X, J = patch.eval_grid(nodes)
        detJ = np.abs(np.linalg.det(J))
    wq = weights[0]
    for w in weights[1:]:
        wq = np.multiply.outer(wq, w)
    T = wq * detJ * problem.source(X)
    for a in range(d):
        T = np.moveaxis(np.asarray(Bd[a].T @ np.moveaxis(T, a, 0).reshape(T.shape[a], -1))
                        .reshape((Bd[a].shape[1],) + tuple(np.delete(T.shape, a))), 0, a)
    return T.ravel()


def assemble_rhs(hier, asm, problem):
    """Finest-level load vector with the Dirichlet lift eliminated (``assembly.py:639-669``)."""
    if asm.level != hier.L:
        raise ValueError("right-hand side is assembled on the finest level only")
    dofs = hier.dofs[hier.L]
    load = np.zeros(dofs.n_block)
    for k in range(hier.domain.num_patches):
        lo, hi = dofs.offsets[k], dofs.offsets[k + 1]
        load[lo:hi] = _tensor_load(hier.spaces[hier.L][k], hier.domain.patches[k], problem)
    fob = dofs.free_of_block
    sel = fob >= 0
    load_free = np.zeros(dofs.n_free)
    np.add.at(load_free, fob[sel], load[sel])
    if dofs.n_dirichlet:
        lift = problem.dirichlet(asm.dirichlet_points)
        load_free = load_free - asm.couple @ lift
    return load_free


def matrix_free_data(hier, level):
    """Sum-factorisation description of the assembled ``A_level`` for the device matrix-free
    operator, or None when it does not apply.  Applies to conforming spaces on patches with a
    constant diagonal Jacobian, exactly the case ``_bulk_matrices`` assembles by Kronecker products
    (``assembly.py:333-344``): per patch K = sum_a c_a (x)_i (K_i if i == a else M_i),
    c_a = det / s_a^2, reduced to free DoFs with shared copies summed."""
    if hier.mode != "conforming" or hier.dim not in (2, 3):
        return None
    dofs = hier.dofs[level]
    d = hier.dim
    bands_M, bands_K, cs = [], [], []
    mats = []
    for k in range(hier.domain.num_patches):
        scal = _probe_jacobian(hier.domain.patches[k])
        if scal is None:
            return None
        det = float(np.prod(scal))
        cs.append([det / scal[a] ** 2 for a in range(d)])
        mats.append([(bs.univariate_mass(s).tocsr(), bs.univariate_stiffness(s).tocsr())
                     for s in hier.spaces[level][k]])
    p = 0
    for per in mats:
        for M, K in per:
            for X in (M, K):
                C = X.tocoo()
                if C.nnz:
                    p = max(p, int(np.abs(C.row - C.col).max()))
    w = 2 * p + 1
    for per in mats:
        for M, K in per:
            for X, out in ((M, bands_M), (K, bands_K)):
                C = X.tocoo()
                band = np.zeros((X.shape[0], w))
                band[C.row, C.col - C.row + p] = C.data
                out.append(band.ravel())
    return dict(dim=d, p=p, dims=np.array([dofs.dims[k] for k in range(hier.domain.num_patches)], dtype=np.int32),
                c=np.array(cs, dtype=np.float64), Mband=np.concatenate(bands_M), Kband=np.concatenate(bands_K),
                block_free=dofs.free_of_block.astype(np.int32))


def check_coercivity(asm):
    """Smallest eigenvalue of the assembled operator (dense diagnostic, ``assembly.py:705-715``);
    a non-positive one means the SIPG penalty sigma is too small."""
    lam = scipy.linalg.eigh(asm.A.toarray(), eigvals_only=True, subset_by_index=[0, 0])[0]
    if lam <= 0:
        raise ValueError(f"assembled operator is not positive definite (lambda_min={lam:.3e}); "
                         "increase the penalty parameter sigma")
    return lam


def geometry_condition_diagnostic(A, A_hat):
    """(lambda_min, lambda_max, ratio) of the pencil (A, A_hat) (``assembly.py:718-723``)."""
    from . import linsolve
    ev = linsolve.dense_generalized_eig(A, A_hat)
    return float(ev[0]), float(ev[-1]), float(ev[-1] / ev[0])


def solution_coefficients(hier, asm, u_free, problem=None):
    """Block-numbered coefficients of a free-DoF vector; with ``problem`` the Dirichlet lift is
    added (``assembly.py:726-733``)."""
    dofs = hier.dofs[asm.level]
    u = np.zeros(dofs.n_block)
    sel = dofs.free_of_block >= 0
    u[sel] = np.asarray(u_free, dtype=float)[dofs.free_of_block[sel]]
    if problem is not None and dofs.n_dirichlet:
        g = problem.dirichlet(asm.dirichlet_points)
        dsel = dofs.dir_of_block >= 0
        u[dsel] += g[dofs.dir_of_block[dsel]]
    return u


def l2_error(hier, asm, u_free, problem):
    """|| u_h - u ||_{L2(Omega)} by Gauss quadrature per patch (``assembly.py:736-755``); a
    diagnostic of the discretisation, not on the solve path."""
    u_block = solution_coefficients(hier, asm, u_free, problem)
    dofs = hier.dofs[asm.level]
    total = 0.0
    for k in range(hier.domain.num_patches):
        spaces = hier.spaces[asm.level][k]
        nodes, weights, Bd = [], [], []
        for sp in spaces:
            x, w = bs.gauss_points(sp)
            nodes.append(x)
            weights.append(w)
            Bd.append(bs.basis_matrices(sp, x, 0)[0])
        X, J = hier.domain.patches[k].eval_grid(nodes)
        wq = weights[0]
        for w in weights[1:]:
            wq = np.multiply.outer(wq, w)
        # u_h on the quadrature grid: contract the coefficient tensor axis by axis
        T = u_block[dofs.offsets[k]:dofs.offsets[k + 1]].reshape(dofs.dims[k])
        for a in range(len(spaces)):
            T = np.moveaxis(np.asarray(Bd[a] @ np.moveaxis(T, a, 0).reshape(T.shape[a], -1))
                            .reshape((Bd[a].shape[0],) + tuple(np.delete(T.shape, a))), 0, a)
        diff = T - problem.exact(X)
        total += float(np.sum(wq * np.abs(np.linalg.det(J)) * diff ** 2))
    return float(np.sqrt(total))


def prolongation(hier, level):
    """Free-DoF embedding of level-1 into level (``assembly.py:672-702``).

    Per patch the Kronecker product of 1-D two-scale matrices; entries of
    shared (interface) DoFs are assigned once, not summed.
    """
    if level < 1:
        raise ValueError("prolongation needs level >= 1")
    dofs_f, dofs_c = hier.dofs[level], hier.dofs[level - 1]
    rows, cols, vals = [], [], []
    for k in range(hier.domain.num_patches):
        mats = []
        for sc, sf in zip(hier.spaces[level - 1][k], hier.spaces[level][k]):
            if sc == sf:
                mats.append(scipy.sparse.identity(sc.n, format="csr"))
            else:
                refined, P1 = bs.two_scale_refine(sc)
                if refined != sf:
                    raise AssertionError("hierarchy spaces are not dyadically nested")
                mats.append(P1)
        r, c, v = _map_coo(_kron_chain(mats), dofs_f.free_of_block, dofs_c.free_of_block,
                           int(dofs_f.offsets[k]), int(dofs_c.offsets[k]))
        rows.append(r)
        cols.append(c)
        vals.append(v)
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    v = np.concatenate(vals)
    key = r * np.int64(dofs_c.n_free) + c
    _, first = np.unique(key, return_index=True)
    return scipy.sparse.csr_matrix((v[first], (r[first], c[first])), shape=(dofs_f.n_free, dofs_c.n_free))


def prolongation_kron(hier, level):
    """Kronecker description of ``prolongation(hier, level)`` for the device transfer.

    The reference builds P per patch as the Kronecker product of 1-D two-scale matrices and
    maps it to free DoFs, assigning (not summing) the rows of shared interface DoFs
    (``assembly.py:672-702``).  Returned here instead of the assembled CSR:

    * ``nf``, ``nc``: int32 [npatch, dim] per-patch block sizes of the fine / coarse level;
    * ``idx``, ``val``: the 1-D matrices P_{k,a} (patch-major, then axis) as ELL rows of
      ``width`` entries (column -1 = padding), row-major;
    * ``fine_free`` / ``coarse_free``: block index -> free id (-1: Dirichlet);
    * ``fine_owner``: 1 where the fine block copy is its class root -- the one copy a
      restriction may read, so that shared rows are counted once as in P^T.
    """
    if level < 1:
        raise ValueError("prolongation needs level >= 1")
    dofs_f, dofs_c = hier.dofs[level], hier.dofs[level - 1]
    npatch = hier.domain.num_patches
    dim = len(hier.spaces[level][0])
    mats = []
    for k in range(npatch):
        for sc, sf in zip(hier.spaces[level - 1][k], hier.spaces[level][k]):
            if sc == sf:
                mats.append(scipy.sparse.identity(sc.n, format="csr"))
            else:
                refined, P1 = bs.two_scale_refine(sc)
                if refined != sf:
                    raise AssertionError("hierarchy spaces are not dyadically nested")
                mats.append(scipy.sparse.csr_matrix(P1))
    width = max(int(np.diff(m.indptr).max()) for m in mats)
    idx, val = [], []
    for m in mats:
        m = scipy.sparse.csr_matrix(m)
        m.sort_indices()
        n = m.shape[0]
        cnt = np.diff(m.indptr)
        slot = np.arange(m.nnz) - np.repeat(m.indptr[:-1], cnt)
        rows = np.repeat(np.arange(n), cnt)
        i2 = np.full((n, width), -1, dtype=np.int32)
        v2 = np.zeros((n, width))
        i2[rows, slot] = m.indices
        v2[rows, slot] = m.data
        idx.append(i2.ravel())
        val.append(v2.ravel())
    nf = np.array([dofs_f.dims[k] for k in range(npatch)], dtype=np.int32).reshape(npatch, dim)
    nc = np.array([dofs_c.dims[k] for k in range(npatch)], dtype=np.int32).reshape(npatch, dim)
    return dict(dim=dim, nf=nf, nc=nc, width=width,
                idx=np.concatenate(idx).astype(np.int32), val=np.concatenate(val),
                fine_free=dofs_f.free_of_block.astype(np.int32),
                fine_owner=(dofs_f.class_of == np.arange(dofs_f.n_block)).astype(np.int32),
                coarse_free=dofs_c.free_of_block.astype(np.int32),
                n_fine=dofs_f.n_free, n_coarse=dofs_c.n_free)


def kron_apply(kd, x, transpose=False):
    """Host restatement of the device Kronecker transfer (test check): P x, or P^T x."""
    dim, npatch = kd["dim"], kd["nf"].shape[0]
    out = np.zeros(kd["n_coarse"] if transpose else kd["n_fine"])
    width = kd["width"]
    pos = 0
    offf = np.concatenate([[0], np.cumsum(np.prod(kd["nf"], axis=1))])
    offc = np.concatenate([[0], np.cumsum(np.prod(kd["nc"], axis=1))])
    for k in range(npatch):
        ops = []
        for a in range(dim):
            n_f, n_c = int(kd["nf"][k, a]), int(kd["nc"][k, a])
            i2 = kd["idx"][pos: pos + n_f * width].reshape(n_f, width)
            v2 = kd["val"][pos: pos + n_f * width].reshape(n_f, width)
            pos += n_f * width
            rows = np.repeat(np.arange(n_f), width)
            m = i2.ravel() >= 0
            ops.append(scipy.sparse.csr_matrix((v2.ravel()[m], (rows[m], i2.ravel()[m])), shape=(n_f, n_c)))
        Pk = _kron_chain(ops)
        ff = kd["fine_free"][offf[k]:offf[k + 1]]
        cf = kd["coarse_free"][offc[k]:offc[k + 1]]
        if transpose:
            own = kd["fine_owner"][offf[k]:offf[k + 1]].astype(bool) & (ff >= 0)
            r = np.zeros(len(ff))
            r[own] = x[ff[own]]
            z = Pk.T @ r
            np.add.at(out, cf[cf >= 0], z[cf >= 0])
        else:
            e = np.where(cf >= 0, x[np.maximum(cf, 0)], 0.0)
            y = Pk @ e
            own = kd["fine_owner"][offf[k]:offf[k + 1]].astype(bool) & (ff >= 0)
            out[ff[own]] = y[own]
    return out
