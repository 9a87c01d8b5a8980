"""ctypes binding of ``libigb_setup.so`` (csrc/host_setup.cpp): native host-setup steps.

Bit-identical replacements of the SciPy steps that dominate the large configurations' setup
(Kronecker assembly of affine patches reduced to free DoFs, the Galerkin product ``P^T A P``,
the assembled operator's symmetry check).  Setup stays on the host, as in the reference; when
the library is absent (``IGB_NATIVE_SETUP=0`` or not built) the SciPy path runs instead and
produces the same arrays (``tests/test_setup.py`` compares both).
"""

import ctypes
import os

import numpy as np
import scipy.sparse

_HERE = os.path.dirname(os.path.abspath(__file__))
_PATH = os.path.join(_HERE, "libigb_setup.so")
_lib = None
_p = ctypes.c_void_p
_i64 = ctypes.c_int64


def lib():
    """The loaded library, or None (not built / disabled with IGB_NATIVE_SETUP=0)."""
    global _lib
    if os.environ.get("IGB_NATIVE_SETUP", "1") == "0":
        return None
    if _lib is None:
        if not os.path.exists(_PATH):
            return None
        L = ctypes.CDLL(_PATH)
        L.igbs_kron_reduce.argtypes = [ctypes.c_int, ctypes.c_int] + [_p] * 11 + [_i64, _i64]
        L.igbs_kron_reduce.restype = _p
        L.igbs_galerkin.argtypes = [_i64, _i64] + [_p] * 6
        L.igbs_galerkin.restype = _p
        L.igbs_nnz.argtypes = [_p]
        L.igbs_nnz.restype = _i64
        L.igbs_copy.argtypes = [_p, _p, ctypes.c_int, _p, _p]
        L.igbs_copy.restype = None
        L.igbs_free.argtypes = [_p]
        L.igbs_free.restype = None
        L.igbs_max_asym.argtypes = [_i64, _p, _p, _p, _p, _p]
        L.igbs_max_asym.restype = None
        _lib = L
    return _lib


def _a(x, dtype):
    return np.ascontiguousarray(x, dtype=dtype)


def _ptr(x):
    return x.ctypes.data_as(_p)


def _take(L, h, shape):
    """Copy a result handle into a scipy CSR (int32 indices, int32 indptr when nnz < 2^31)."""
    try:
        nnz = int(L.igbs_nnz(h))
        idx64 = nnz >= 2 ** 31 - 1
        indptr = np.empty(shape[0] + 1, dtype=np.int64 if idx64 else np.int32)
        indices = np.empty(nnz, dtype=np.int32)
        data = np.empty(nnz, dtype=np.float64)
        L.igbs_copy(h, _ptr(indptr), 1 if idx64 else 0, _ptr(indices), _ptr(data))
    finally:
        L.igbs_free(h)
    out = scipy.sparse.csr_matrix((data, indices, indptr), shape=shape)
    out.has_sorted_indices = True
    return out


def kron_reduce(dims, coef, oned, block_off, row_map, col_map, n_rows, n_cols):
    """Free-DoF CSR of sum_k sum_a coef[k,a] (x)_i (K if i == a else M)_{k,i}, rows / columns mapped
    through row_map / col_map (-1 dropped), SciPy's COO -> CSR summation order.

    oned[k][a] = (M, K) 1-D CSR matrices of patch k, axis a, with identical sorted patterns.
    Returns None when the library is unavailable."""
    L = lib()
    if L is None:
        return None
    npatch, dim = len(dims), len(dims[0])
    ptrs, idxs, mv, kv, ptr_off, ent_off = [], [], [], [], [], []
    po = eo = 0
    for k in range(npatch):
        for a in range(dim):
            M, K = oned[k][a]
            ptrs.append(_a(M.indptr, np.int32))
            idxs.append(_a(M.indices, np.int32))
            mv.append(_a(M.data, np.float64))
            kv.append(_a(K.data, np.float64))
            ptr_off.append(po)
            ent_off.append(eo)
            po += len(M.indptr)
            eo += len(M.indices)
    ip, ix = np.concatenate(ptrs), np.concatenate(idxs)
    mval, kval = np.concatenate(mv), np.concatenate(kv)
    d = _a(dims, np.int32).ravel()
    c = _a(coef, np.float64).ravel()
    bo = _a(block_off, np.int64)
    po_a, eo_a = _a(ptr_off, np.int64), _a(ent_off, np.int64)
    rm, cm = _a(row_map, np.int32), _a(col_map, np.int32)
    h = L.igbs_kron_reduce(dim, npatch, _ptr(bo), _ptr(d), _ptr(c), _ptr(po_a), _ptr(eo_a), _ptr(ip), _ptr(ix),
                           _ptr(mval), _ptr(kval), _ptr(rm), _ptr(cm), int(n_rows), int(n_cols))
    return _take(L, h, (int(n_rows), int(n_cols)))


def galerkin(A, P):
    """(P^T A) P with SciPy's csc_matmat arithmetic, as sorted CSR; None without the library."""
    L = lib()
    if L is None:
        return None
    A = A.tocsr()
    P = P.tocsr()
    if not A.has_sorted_indices:
        A = A.sorted_indices()
    if not P.has_sorted_indices:
        P = P.sorted_indices()
    nf, nc = P.shape
    ap, ai, av = _a(A.indptr, np.int64), _a(A.indices, np.int32), _a(A.data, np.float64)
    pp, pi, pv = _a(P.indptr, np.int64), _a(P.indices, np.int32), _a(P.data, np.float64)
    h = L.igbs_galerkin(nf, nc, _ptr(ap), _ptr(ai), _ptr(av), _ptr(pp), _ptr(pi), _ptr(pv))
    return _take(L, h, (nc, nc))


def max_asym(A):
    """(max |A - A^T|, max |A|) over the stored pattern; None without the library."""
    L = lib()
    if L is None:
        return None
    A = A.tocsr()
    if not A.has_sorted_indices:
        A = A.sorted_indices()
    ap, ai, av = _a(A.indptr, np.int64), _a(A.indices, np.int32), _a(A.data, np.float64)
    a, b = ctypes.c_double(), ctypes.c_double()
    L.igbs_max_asym(A.shape[0], _ptr(ap), _ptr(ai), _ptr(av), ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value
