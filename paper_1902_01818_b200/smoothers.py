"""Smoother setup: Gauss-Seidel, subspace-corrected mass (SCMS) and hybrid.

Public surface of the reference's ``igamg.smoothers`` (``smoothers.py:23-32``).
Construction (piece decomposition, 1-D generalized eigenproblems, interface
piece inverses) stays on the host, as in the reference; the *application* of
every smoother runs on the device through ``libigb`` once the owning
:class:`~paper_1902_01818_b200.multigrid.MultigridSolver` has uploaded the
level (``bind``).  There is no host implementation of the apply paths.

Device data produced here:

* ``ScmsInteriorSolver.square_transforms`` / ``denominator`` -- the sum over
  the 2^d subspaces of the reference's fast diagonalisation
  (``smoothers.py:283-294``) equals one square-transform FD
  ``X = T (T^T R T ./ D) T^T`` with ``T_a = [W_L V_L | W_C V_C]``; ``D`` is the
  subspace denominators assembled block-wise.
* ``SubspaceCorrectedMass.piece_inverses`` -- dense inverses of the interface
  principal submatrices, obtained column by column from the same SuperLU
  factorization the reference builds (``smoothers.py:316-319``).
"""

from dataclasses import dataclass, field

import os

import numpy as np
import scipy.linalg
import scipy.sparse

from . import bspline as bs
from . import linsolve

__all__ = [
    "Piece",
    "PieceDecomposition",
    "build_piece_decomposition",
    "GaussSeidel",
    "gs_apply_forward",
    "gs_apply_backward",
    "ScmsInteriorSolver",
    "SubspaceCorrectedMass",
    "HybridSmoother",
    "build_smoother",
]


@dataclass(frozen=True)
class Piece:
    kind: str  # 'interior' | 'face' | 'edge' | 'vertex'
    indices: np.ndarray = field(repr=False)
    patches: tuple
    entity: tuple

    @property
    def size(self):
        return len(self.indices)


@dataclass
class PieceDecomposition:
    pieces: list
    n_free: int
    interior_dims: dict = field(default_factory=dict)

    def validate_partition(self):
        seen = np.zeros(self.n_free, dtype=np.int64)
        for piece in self.pieces:
            np.add.at(seen, piece.indices, 1)
        if np.any(seen > 1):
            raise AssertionError("piece decomposition is not disjoint")
        if np.any(seen == 0):
            raise AssertionError("piece decomposition does not cover all free dofs")


class _VertexRegistry:
    """Stable ids for geometric points (first-come numbering on a 1e-6 grid)."""

    def __init__(self, tol=1e-6):
        self.tol = tol
        self._ids = {}

    def vertex_id(self, point):
        key = tuple(np.round(np.asarray(point) / self.tol).astype(np.int64))
        return self._ids.setdefault(key, len(self._ids))


def build_piece_decomposition(hier, level):
    """Classify free DoFs by their number of extremal directions (``smoothers.py:83-165``).

    interior = 0 extremal directions; 1 -> edge (2-D) / face (3-D) piece of the
    interface the side belongs to; 2 in 3-D -> geometric edge; d -> vertex.
    Each free DoF is classified by its class root (smallest block index).
    """
    domain = hier.domain
    dofs = hier.dofs[level]
    d = hier.dim
    n_free = dofs.n_free
    rep = dofs.free_representatives()
    k_of = dofs.patch_of_block(rep)
    local = rep - dofs.offsets[k_of]
    multi = np.empty((n_free, d), dtype=np.int64)
    dims_of = np.empty((n_free, d), dtype=np.int64)
    for k in range(domain.num_patches):
        sel = k_of == k
        if np.any(sel):
            multi[sel] = np.stack(np.unravel_index(local[sel], dofs.dims[k]), axis=1)
            dims_of[sel] = dofs.dims[k]
    at_hi = multi == dims_of - 1
    ext = (multi == 0) | at_hi
    m = ext.sum(axis=1)

    side_iface = {}
    for idx, iface in enumerate(domain.interfaces):
        side_iface[(iface.k, iface.side_k.axis, iface.side_k.end)] = idx
        side_iface[(iface.l, iface.side_l.axis, iface.side_l.end)] = idx

    groups = {}
    # one extremal direction: side of an interface
    one = np.flatnonzero(m == 1)
    if len(one):
        axis = np.argmax(ext[one], axis=1)
        end = at_hi[one, axis].astype(np.int64)
        kind = "face" if d == 3 else "edge"
        keys = k_of[one] * (2 * d) + axis * 2 + end
        for key in np.unique(keys):
            k, rem = divmod(int(key), 2 * d)
            a, e = divmod(rem, 2)
            iface_idx = side_iface.get((k, a, e))
            if iface_idx is None:
                raise AssertionError(f"free dof of patch {k} extremal towards a boundary side")
            groups.setdefault((kind, iface_idx), []).append(one[keys == key])
    # vertices and 3-D edges: registry order follows ascending free id
    registry = _VertexRegistry()
    corner_cache = {}

    def corner(k, bits):
        key = (k, tuple(bits))
        if key not in corner_cache:
            corner_cache[key] = domain.patches[k].corner(bits)
        return corner_cache[key]

    special = np.flatnonzero((m == d) | ((d == 3) & (m == 2)))
    for fid in special.tolist():
        k = int(k_of[fid])
        if m[fid] == d:
            bits = tuple(int(b) for b in at_hi[fid])
            entity = ("vertex", registry.vertex_id(corner(k, bits)))
        else:
            ex = np.flatnonzero(ext[fid])
            run = next(a for a in range(d) if a not in ex)
            lo_bits = [0] * d
            hi_bits = [0] * d
            for a in ex:
                lo_bits[a] = hi_bits[a] = int(at_hi[fid, a])
            hi_bits[run] = 1
            v0 = registry.vertex_id(corner(k, lo_bits))
            v1 = registry.vertex_id(corner(k, hi_bits))
            entity = ("edge", tuple(sorted((v0, v1))))
        groups.setdefault(entity, []).append(np.array([fid]))

    pieces = []
    interior_dims = {}
    interior_mask = m == 0
    for k in range(domain.num_patches):
        dims = dofs.dims[k]
        if any(n <= 2 for n in dims):
            continue
        grids = np.meshgrid(*[np.arange(1, n - 1) for n in dims], indexing="ij")
        flat = np.ravel_multi_index([g.ravel() for g in grids], dims)
        ids = dofs.free_of_block[dofs.offsets[k] + flat]
        expected = np.flatnonzero(interior_mask & (k_of == k))
        if not np.array_equal(np.sort(ids), expected):
            raise AssertionError("interior piece does not match the classification")
        interior_dims[k] = tuple(n - 2 for n in dims)
        pieces.append(Piece("interior", ids.astype(np.int64), (k,), ("interior", k)))

    fob = dofs.free_of_block
    blk_patch = dofs.patch_of_block(np.arange(dofs.n_block))
    kind_order = {"face": 0, "edge": 1, "vertex": 2}
    for entity in sorted(groups, key=lambda e: (kind_order[e[0]], str(e[1]))):
        fids = np.sort(np.concatenate(groups[entity])).astype(np.int64)
        member = np.zeros(n_free + 1, dtype=bool)
        member[fids] = True
        sel = member[np.where(fob >= 0, fob, n_free)]
        patch_set = tuple(int(p) for p in np.unique(blk_patch[sel]))
        pieces.append(Piece(entity[0], fids, patch_set, entity))

    deco = PieceDecomposition(pieces, n_free, interior_dims)
    deco.validate_partition()
    return deco


# -- Gauss-Seidel ------------------------------------------------------------------


class _DeviceBound:
    """Mixin: the apply paths run on the device of the owning solver."""

    _ctx = None
    _level = None

    def bind(self, ctx, level):
        self._ctx = ctx
        self._level = level
        return self

    def _require(self):
        if self._ctx is None:
            raise RuntimeError(
                "smoother not bound to a device context; build it through MultigridSolver "
                "(there is no host implementation)")
        return self._ctx

    # smoother duck type of the reference (smoothers.py:192-200, 327-332, 343-353): the steps run
    # on the device (igb_smooth); A must be the level operator the smoother was built for
    _kind = None

    def _smooth(self, A, u, f, steps, post):
        ctx = self._ctx_for_smooth()
        if A is not None and A.shape[0] != len(u):
            raise ValueError("operator and iterate sizes differ")
        out = ctx.smooth(self._level, self._kind, post, steps, f, u)
        u[...] = out  # in place, as the reference's u += ...
        return u

    def _ctx_for_smooth(self):
        return self._require()

    def pre_smooth(self, A, u, f, steps):
        return self._smooth(A, u, f, steps, False)

    def post_smooth(self, A, u, f, steps):
        return self._smooth(A, u, f, steps, True)


class GaussSeidel(_DeviceBound):
    """Forward/backward Gauss-Seidel in natural order (``smoothers.py:171-200``).

    Host setup only validates the diagonal; the level schedules of tril(A)
    and triu(A) are built natively by ``igb_set_gs``.
    """

    _kind = "gs"

    def _ctx_for_smooth(self):
        return self._standalone()

    def __init__(self, A):
        A = A.tocsr()
        if np.any(A.diagonal() == 0.0):
            raise ValueError("Gauss-Seidel needs a nonzero diagonal")
        self.n = A.shape[0]
        self._A = A

    def _standalone(self):
        """A smoother built outside a MultigridSolver (e.g. ``gs_apply_forward(A, r)``) gets its own
        one-level device context: A on level 1 under a trivial 1x1 level 0 (still the device
        sweep; there is no host implementation)."""
        if self._ctx is None:
            from ._lib import Context
            one = scipy.sparse.csr_matrix(np.ones((1, 1)))
            ctx = Context()
            ctx.set_num_levels(1)
            ctx.set_level_matrix(0, one)
            ctx.set_level_matrix(1, self._A)
            ctx.set_prolongation(1, scipy.sparse.csr_matrix(([0.0], ([0], [0])), shape=(self.n, 1)))
            ctx.set_gs(1)
            ctx.set_coarse_lu(one, one, np.zeros(1, np.int32), np.zeros(1, np.int32))
            ctx.set_cycle("gs", 1, np.ones(2, np.int32))
            ctx.finalize()
            self._own_ctx = ctx
            self.bind(ctx, 1)
        return self._ctx

    def apply_forward(self, r):
        return self._standalone().op("gs_fwd", self._level, r, self.n)

    def apply_backward(self, r):
        return self._standalone().op("gs_bwd", self._level, r, self.n)


def gs_apply_forward(A, r):
    """One forward Gauss-Seidel sweep from zero (``smoothers.py:203-204``), on the device."""
    return GaussSeidel(A).apply_forward(r)


def gs_apply_backward(A, r):
    """One backward Gauss-Seidel sweep from zero (``smoothers.py:207-208``), on the device."""
    return GaussSeidel(A).apply_backward(r)


# -- subspace corrected mass ----------------------------------------------------------


class ScmsInteriorSolver:
    """Tensor fast-diagonalisation data of one patch interior (``smoothers.py:203-281``).

    ``_subspaces`` is the reference's list of ``(Ts, denom)`` per subspace
    combination; ``square_transforms`` / ``denominator`` is the equivalent
    single transform used by the device kernels.
    """

    def __init__(self, spaces, delta, interior_policy="product"):
        if delta <= 0:
            raise ValueError("scaling parameter delta must be positive")
        d = len(spaces)
        h = max(s.meshsize for s in spaces)
        self.sigma_scal = 1.0 / (delta * h * h)
        self.dims = tuple(s.n - 2 for s in spaces)
        self.policy = interior_policy
        bases = []
        for s in spaces:
            M = bs.interior_matrix(bs.univariate_mass(s).toarray())
            K = bs.interior_matrix(bs.univariate_stiffness(s).toarray())
            split = bs.reduced_split(s)
            per = []
            for is_large, W in ((True, split.large), (False, split.complement)):
                if W.shape[1] == 0:
                    per.append(None)
                    continue
                lam, V = scipy.linalg.eigh(W.T @ K @ W, W.T @ M @ W)
                if is_large and interior_policy == "surrogate":
                    lam = np.full_like(lam, self.sigma_scal)
                elif is_large and interior_policy == "mass":
                    lam = np.zeros_like(lam)
                elif is_large and interior_policy == "bound":
                    lam = np.full_like(lam, lam[-1])
                per.append((W @ V, lam))
            bases.append(per)
        self._bases = bases
        self._subspaces = []
        self._alphas = []
        for alpha in np.ndindex(*(2,) * d):
            if any(bases[a][alpha[a]] is None for a in range(d)):
                continue
            Ts = [bases[a][alpha[a]][0] for a in range(d)]
            self._subspaces.append((Ts, self._subspace_denom(alpha)))
            self._alphas.append(alpha)
        self._square = None

    def _subspace_denom(self, alpha):
        d = len(alpha)
        lams = [self._bases[a][alpha[a]][1] for a in range(d)]
        if self.policy == "product":
            denom = lams[0] + self.sigma_scal
            for a in range(1, d):
                denom = np.multiply.outer(denom, lams[a] + self.sigma_scal)
            return denom / self.sigma_scal ** (d - 1)
        lam = lams[0]
        for a in range(1, d):
            lam = np.add.outer(lam, lams[a])
        return lam if self.policy == "surrogate" else lam + self.sigma_scal

    def _build_square(self):
        d = len(self.dims)
        Ts, offs = [], []
        for a in range(d):
            blocks = [b[0] for b in self._bases[a] if b is not None]
            Ts.append(np.ascontiguousarray(np.hstack(blocks)))
            sizes = [b[0].shape[1] if b is not None else 0 for b in self._bases[a]]
            offs.append((0, sizes[0], sizes[0] + sizes[1]))
        D = np.zeros(self.dims)
        for alpha, (_, denom) in zip(self._alphas, self._subspaces):
            sl = tuple(slice(offs[a][alpha[a]], offs[a][alpha[a] + 1]) for a in range(d))
            D[sl] = denom
        self._square = (Ts, np.ascontiguousarray(D))

    @property
    def square_transforms(self):
        if self._square is None:
            self._build_square()
        return self._square[0]

    @property
    def denominator(self):
        if self._square is None:
            self._build_square()
        return self._square[1]


def _tensor_face(sub, piece, hier, level, tol=1e-13, nmax=160):
    """Fast diagonalisation of a 3-D face piece, when its matrix has the tensor form.

    The reference solves every interface piece with SuperLU on the principal submatrix
    ``A[idx][:, idx]`` (``smoothers.py:316-319``).  On conforming affine patches the face between
    two patches is a 2-D tensor grid and that submatrix is
        a M1 (x) M2 + b1 K1 (x) M2 + b2 M1 (x) K2
    (M_i, K_i: interior blocks of the tangential 1-D mass / stiffness matrices; a, b_i collect the
    normal direction's boundary entries of both patches).  Then, with K_i V_i = M_i V_i L_i and
    V_i^T M_i V_i = I,
        sub^-1 R = V1 ((V1^T R V2) ./ (a + b1 l1_j + b2 l2_k)) V2^T,
    which the device applies with the interiors' 2-D kernels instead of streaming a dense m x m
    inverse (cfg5: twelve 4225^2 inverses = 1.7 GB per application).  The form is *fitted and
    verified numerically* (max |sub - fit| <= tol max |sub|); anything else keeps the dense
    inverse.  Returns (dims, [V1, V2], denominator) or None."""
    import scipy.linalg as sla
    import scipy.sparse as sp
    from . import bspline
    if hier.dim != 3 or piece.kind != "face":
        return None
    iface = hier.domain.interfaces[piece.entity[1]]
    k, axis = iface.k, iface.side_k.axis
    spaces = hier.spaces[level][k]
    tang = [a for a in range(3) if a != axis]
    Ms = [bspline.interior_matrix(bspline.univariate_mass(spaces[a])).tocsr() for a in tang]
    Ks = [bspline.interior_matrix(bspline.univariate_stiffness(spaces[a])).tocsr() for a in tang]
    dims = tuple(M.shape[0] for M in Ms)
    if dims[0] * dims[1] != sub.shape[0] or max(dims) > nmax or min(dims) < 1:
        return None
    basis = [sp.kron(Ms[0], Ms[1], format="csr"), sp.kron(Ks[0], Ms[1], format="csr"),
             sp.kron(Ms[0], Ks[1], format="csr")]
    S = sub.tocsr()
    G = np.array([[bi.multiply(bj).sum() for bj in basis] for bi in basis])
    rhs = np.array([bi.multiply(S).sum() for bi in basis])
    try:
        coef = np.linalg.solve(G, rhs)
    except np.linalg.LinAlgError:
        return None
    fit = coef[0] * basis[0] + coef[1] * basis[1] + coef[2] * basis[2]
    err = abs(S - fit).max()
    if not err <= tol * abs(S).max():
        return None
    lam, V = [], []
    for M, K in zip(Ms, Ks):
        w, v = sla.eigh(K.toarray(), M.toarray())
        lam.append(w)
        V.append(np.ascontiguousarray(v))
    denom = coef[0] + coef[1] * lam[0][:, None] + coef[2] * lam[1][None, :]
    if not np.all(denom > 0):
        return None
    return dims, V, np.ascontiguousarray(denom)


class SubspaceCorrectedMass(_DeviceBound):
    """Damped additive piece-local solves of one level (``smoothers.py:297-332``)."""

    _kind = "scms"

    def __init__(self, A, hier, level, tau, delta, interior_policy="product"):
        if tau <= 0 or delta <= 0:
            raise ValueError("scms needs positive damping and scaling")
        self.tau = tau
        self.n = A.shape[0]
        self.decomposition = build_piece_decomposition(hier, level)
        self.interiors = []      # (piece, ScmsInteriorSolver)
        self.pieces = []         # (piece, Factorization)
        self.tensor_faces = {}   # index into pieces -> (dims, [V1, V2], denominator): see _tensor_face
        cache = {}
        A = A.tocsr()
        for piece in self.decomposition.pieces:
            if piece.kind == "interior":
                k = piece.patches[0]
                spaces = hier.spaces[level][k]
                key = (tuple(hash(s) for s in spaces), delta, interior_policy)
                if key not in cache:
                    cache[key] = ScmsInteriorSolver(spaces, delta, interior_policy)
                self.interiors.append((piece, cache[key]))
            else:
                sub = A[piece.indices][:, piece.indices].tocsc()
                self.pieces.append((piece, linsolve.factorize(sub, spd=True)))
                if os.environ.get("IGB_TENSOR_FACES", "1") != "0":
                    fd = _tensor_face(sub, piece, hier, level)
                    if fd is not None:
                        self.tensor_faces[len(self.pieces) - 1] = fd
        self._inverses = None

    @property
    def piece_inverses(self):
        """Dense inverses of the interface principal submatrices (from the SuperLU factors); None for
        the faces applied by fast diagonalisation (``tensor_faces``)."""
        if self._inverses is None:
            dense = [i for i in range(len(self.pieces)) if i not in self.tensor_faces]
            inv = linsolve.inverses([self.pieces[i][1] for i in dense])
            self._inverses = [None] * len(self.pieces)
            for i, m in zip(dense, inv):
                self._inverses[i] = m
        return self._inverses

    def apply(self, r):
        return self._require().op("scms", self._level, r, self.n)


class HybridSmoother:
    """Forward GS then SCMS steps before coarsening, mirrored afterwards (``smoothers.py:335-353``)."""

    def __init__(self, gs, scms, nu_inner=1):
        self.gs = gs
        self.scms = scms
        self.nu_inner = nu_inner

    def bind(self, ctx, level):
        self.gs.bind(ctx, level)
        self.scms.bind(ctx, level)
        return self

    def pre_smooth(self, A, u, f, steps):
        """GS forward, then steps * nu_inner SCMS steps (``smoothers.py:343-347``), on the device."""
        out = self.scms._require().smooth(self.scms._level, "hyb", False, steps * self.nu_inner, f, u)
        u[...] = out
        return u

    def post_smooth(self, A, u, f, steps):
        """steps * nu_inner SCMS steps, then GS backward (``smoothers.py:349-353``), on the device."""
        out = self.scms._require().smooth(self.scms._level, "hyb", True, steps * self.nu_inner, f, u)
        u[...] = out
        return u


def build_smoother(kind, A, hier, level, tau=1.0, delta=0.12, interior_policy="product"):
    if kind == "gs":
        return GaussSeidel(A)
    if kind == "scms":
        return SubspaceCorrectedMass(A, hier, level, tau, delta, interior_policy)
    if kind == "hyb":
        return HybridSmoother(GaussSeidel(A),
                              SubspaceCorrectedMass(A, hier, level, tau, delta, interior_policy))
    raise ValueError(f"unknown smoother kind {kind!r}")
