"""ctypes binding of ``libigb.so`` (the C ABI in ``include/igb.h``).

There is no CPU fallback: if the shared library is missing or no CUDA device
is usable, constructing a :class:`Context` raises ``RuntimeError``.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IGB_LIB", os.path.join(_HERE, "libigb.so"))

OP = {
    "spmv": 0, "residual": 1, "gs_fwd": 2, "gs_bwd": 3, "scms": 4,
    "restrict": 5, "prolong": 6, "coarse": 7, "cycle": 8,
}
SMOOTHER = {"gs": 0, "scms": 1, "hyb": 2}
KERNEL_CLASSES = ("spmv", "gs", "fd", "pieces", "transfer", "coarse", "cg")

# Every exported symbol with its ctypes signature (argtypes, restype).
_i, _ll, _d = ctypes.c_int, ctypes.c_longlong, ctypes.c_double
_p = ctypes.c_void_p
_ip = ctypes.POINTER(ctypes.c_int)
SIGNATURES = {
    "igb_version": ([], _i),
    "igb_create": ([ctypes.POINTER(_p), _i], _i),
    "igb_destroy": ([_p], _i),
    "igb_last_error": ([_p], ctypes.c_char_p),
    "igb_set_num_levels": ([_p, _i], _i),
    "igb_set_level_matrix": ([_p, _i, _i, _ll, _p, _p, _p], _i),
    "igb_set_prolongation": ([_p, _i, _i, _i, _ll, _p, _p, _p], _i),
    "igb_set_prolongation_kron": ([_p, _i, _i, _i, _p, _p, _i, _p, _p, _p, _p, _p], _i),
    "igb_set_matrix_free": ([_p, _i, _i, _i, _i, _p, _p, _p, _p, _p], _i),
    "igb_set_gs": ([_p, _i], _i),
    "igb_scms_begin": ([_p, _i, _d], _i),
    "igb_scms_add_interior": ([_p, _i, _i, _p, _p, _p, _p, _p, _p], _i),
    "igb_scms_add_piece": ([_p, _i, _i, _p, _p], _i),
    "igb_set_coarse_lu": ([_p, _i, _ll, _p, _p, _p, _ll, _p, _p, _p, _p, _p], _i),
    "igb_set_cycle": ([_p, _i, _i, _p], _i),
    "igb_finalize": ([_p], _i),
    "igb_cycle": ([_p, _i, _p, _p], _i),
    "igb_op": ([_p, _i, _i, _p, _p], _i),
    "igb_pcg": ([_p, _p, _d, _i, _p, _ip, _p, _i], _i),
    "igb_pcg_device": ([_p, _p, _d, _i, _p, _ip, _p, _i], _i),
    "igb_device_alloc": ([_p, _ll, ctypes.POINTER(_p)], _i),
    "igb_host_alloc": ([_p, _ll, ctypes.POINTER(_p)], _i),
    "igb_host_free": ([_p, _p], _i),
    "igb_device_free": ([_p, _p], _i),
    "igb_memcpy_h2d": ([_p, _p, _p, _ll], _i),
    "igb_memcpy_d2h": ([_p, _p, _p, _ll], _i),
    "igb_last_timing": ([_p, ctypes.POINTER(_d), ctypes.POINTER(_d)], _i),
    "igb_launch_count": ([_p, ctypes.POINTER(_ll), _i], _i),
    "igb_profile_enable": ([_p, _i], _i),
    "igb_profile_reset": ([_p], _i),
    "igb_profile_get": ([_p, _i, ctypes.POINTER(_d), ctypes.POINTER(_ll), ctypes.POINTER(_d)], _i),
    "igb_gs_info": ([_p, _i, _i, _ip, _i], _i),
    "igb_smooth": ([_p, _i, _i, _i, _i, _p, _p], _i),
    "igb_cg": ([_p, _i, _ll, _p, _p, _p, _i, _p, _p, _p, _p, _p, _d, _i, _p, _ip, _p, _i], _i),
    "igb_profile_flops": ([_p, _i, ctypes.POINTER(_d)], _i),
    "igb_profile_top": ([_p, _i, ctypes.POINTER(_d), ctypes.POINTER(_ll), ctypes.POINTER(_d)], _i),
}
PREC = {"none": 0, "cycle": 1, "host": 2}
PREC_FN = ctypes.CFUNCTYPE(None, ctypes.POINTER(_d), ctypes.POINTER(_d), _i, _p)
ITER_FN = ctypes.CFUNCTYPE(None, _i, _d, _p)
GS_ENGINES = {1: "panel", 2: "flow", 3: "levelset", 4: "schedule", 5: "line", 6: "wave"}

_lib = None


def load():
    """Load libigb.so once; raises RuntimeError when it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libigb.so not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class IgbError(RuntimeError):
    pass


class Context:
    """Owns one ``igb_ctx`` (one CUDA stream + all device buffers of a hierarchy)."""

    def __init__(self, device=0):
        self.lib = load()
        h = ctypes.c_void_p()
        rc = self.lib.igb_create(ctypes.byref(h), int(device))
        if rc != 0:
            raise RuntimeError(f"igb_create failed ({rc}): no usable CUDA device {device}")
        self.h = h
        self._keep = []

    def _check(self, rc, what):
        if rc != 0:
            msg = self.lib.igb_last_error(self.h).decode()
            raise IgbError(f"{what} failed ({rc}): {msg}")

    def close(self):
        if getattr(self, "h", None):
            for p in getattr(self, "_pinned", []):
                self.lib.igb_host_free(self.h, ctypes.c_void_p(p))
            self._pinned = []
            self.lib.igb_destroy(self.h)
            self.h = None

    def pinned(self, n):
        """float64[n] numpy array in page-locked host memory (freed with the context): host
        buffers for ``pcg`` that copy at full link speed."""
        p = ctypes.c_void_p()
        self._check(self.lib.igb_host_alloc(self.h, 8 * max(1, int(n)), ctypes.byref(p)), "igb_host_alloc")
        if not hasattr(self, "_pinned"):
            self._pinned = []
        self._pinned.append(p.value)
        return np.frombuffer((ctypes.c_double * max(1, int(n))).from_address(p.value), dtype=np.float64)[:int(n)]

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- setup ---------------------------------------------------------------
    def set_num_levels(self, L):
        self._check(self.lib.igb_set_num_levels(self.h, int(L)), "igb_set_num_levels")

    @staticmethod
    def _csr_arrays(M):
        M = M.tocsr()
        M.sort_indices()
        return (_c(M.indptr, np.int32), _c(M.indices, np.int32), _c(M.data, np.float64))

    def set_level_matrix(self, level, A):
        p, i, v = self._csr_arrays(A)
        self._check(self.lib.igb_set_level_matrix(self.h, level, A.shape[0], len(v), _ptr(p), _ptr(i), _ptr(v)),
                    "igb_set_level_matrix")

    def set_prolongation(self, level, P):
        p, i, v = self._csr_arrays(P)
        self._check(self.lib.igb_set_prolongation(self.h, level, P.shape[0], P.shape[1], len(v),
                                                  _ptr(p), _ptr(i), _ptr(v)), "igb_set_prolongation")

    def set_prolongation_kron(self, level, kd):
        """Kronecker form of P_level (assembly.prolongation_kron)."""
        arrs = [_c(kd[k], np.int32) for k in ("nf", "nc", "idx")] + [_c(kd["val"], np.float64)] + \
               [_c(kd[k], np.int32) for k in ("fine_free", "fine_owner", "coarse_free")]
        nf, nc, idx, val, ff, fo, cf = arrs
        self._check(self.lib.igb_set_prolongation_kron(self.h, level, int(kd["dim"]), int(kd["nf"].shape[0]),
                                                       _ptr(nf), _ptr(nc), int(kd["width"]), _ptr(idx), _ptr(val),
                                                       _ptr(ff), _ptr(fo), _ptr(cf)),
                    "igb_set_prolongation_kron")

    def set_matrix_free(self, level, md):
        """Matrix-free form of A_level (assembly.matrix_free_data)."""
        dims, c = _c(md["dims"], np.int32), _c(md["c"], np.float64)
        Mb, Kb, bf = _c(md["Mband"], np.float64), _c(md["Kband"], np.float64), _c(md["block_free"], np.int32)
        self._check(self.lib.igb_set_matrix_free(self.h, level, int(md["dim"]), int(dims.shape[0]), int(md["p"]),
                                                 _ptr(dims), _ptr(c), _ptr(Mb), _ptr(Kb), _ptr(bf)),
                    "igb_set_matrix_free")

    def set_gs(self, level):
        self._check(self.lib.igb_set_gs(self.h, level), "igb_set_gs")

    def scms_begin(self, level, tau):
        self._check(self.lib.igb_scms_begin(self.h, level, float(tau)), "igb_scms_begin")

    def scms_add_interior(self, level, dims, Ts, denom, idx):
        dims_a = _c(dims, np.int32)
        Ts = [_c(T, np.float64) for T in Ts]
        denom = _c(denom, np.float64)
        idx = _c(idx, np.int32)
        # keep the transform arrays alive: the library de-duplicates uploads by host address
        self._keep.extend(Ts + [denom])
        T2 = Ts[2] if len(Ts) > 2 else None
        self._check(self.lib.igb_scms_add_interior(self.h, level, len(dims), _ptr(dims_a), _ptr(Ts[0]),
                                                   _ptr(Ts[1]), _ptr(T2), _ptr(denom), _ptr(idx)),
                    "igb_scms_add_interior")

    def scms_add_piece(self, level, idx, inv):
        idx = _c(idx, np.int32)
        inv = _c(inv, np.float64)
        self._check(self.lib.igb_scms_add_piece(self.h, level, len(idx), _ptr(idx), _ptr(inv)),
                    "igb_scms_add_piece")

    def set_coarse_lu(self, L, U, perm_r, perm_c):
        lp, li, lv = self._csr_arrays(L)
        up, ui, uv = self._csr_arrays(U)
        pr, pc = _c(perm_r, np.int32), _c(perm_c, np.int32)
        self._check(self.lib.igb_set_coarse_lu(self.h, L.shape[0], len(lv), _ptr(lp), _ptr(li), _ptr(lv),
                                               len(uv), _ptr(up), _ptr(ui), _ptr(uv), _ptr(pr), _ptr(pc)),
                    "igb_set_coarse_lu")

    def set_cycle(self, smoother, mu, steps):
        st = _c(steps, np.int32)
        self._check(self.lib.igb_set_cycle(self.h, SMOOTHER[smoother], int(mu), _ptr(st)), "igb_set_cycle")

    def finalize(self):
        self._check(self.lib.igb_finalize(self.h), "igb_finalize")

    # -- compute -------------------------------------------------------------
    def op(self, name, level, x, out_len, out_init=None):
        x = _c(x, np.float64)
        out = np.empty(out_len) if out_init is None else _c(out_init, np.float64).copy()
        self._check(self.lib.igb_op(self.h, OP[name], int(level), _ptr(x), _ptr(out)), f"igb_op({name})")
        return out

    def cycle(self, level, f):
        f = _c(f, np.float64)
        u = np.empty_like(f)
        self._check(self.lib.igb_cycle(self.h, int(level), _ptr(f), _ptr(u)), "igb_cycle")
        return u

    def pcg(self, b, tol, max_iters, out=None):
        """igb_pcg with host buffers; ``out`` (e.g. ``pinned(n)``) receives x."""
        b = _c(b, np.float64)
        x = out if out is not None else np.empty_like(b)
        hist = np.empty(max(1, int(max_iters)))
        its = ctypes.c_int(0)
        self._check(self.lib.igb_pcg(self.h, _ptr(b), float(tol), int(max_iters), _ptr(x), ctypes.byref(its),
                                     _ptr(hist), len(hist)), "igb_pcg")
        n = its.value
        return x, n, hist[:n].tolist()

    def pcg_device(self, d_b, d_x, tol, max_iters):
        hist = np.empty(max(1, int(max_iters)))
        its = ctypes.c_int(0)
        self._check(self.lib.igb_pcg_device(self.h, ctypes.c_void_p(d_b), float(tol), int(max_iters),
                                            ctypes.c_void_p(d_x), ctypes.byref(its), _ptr(hist), len(hist)),
                    "igb_pcg_device")
        return its.value, hist[:its.value].tolist()

    def device_alloc(self, nbytes):
        p = ctypes.c_void_p()
        self._check(self.lib.igb_device_alloc(self.h, int(nbytes), ctypes.byref(p)), "igb_device_alloc")
        return p.value

    def device_free(self, p):
        self._check(self.lib.igb_device_free(self.h, ctypes.c_void_p(p)), "igb_device_free")

    def h2d(self, dptr, arr):
        arr = _c(arr, arr.dtype)
        self._check(self.lib.igb_memcpy_h2d(self.h, ctypes.c_void_p(dptr), _ptr(arr), arr.nbytes), "h2d")

    def d2h(self, arr, dptr):
        self._check(self.lib.igb_memcpy_d2h(self.h, _ptr(arr), ctypes.c_void_p(dptr), arr.nbytes), "d2h")
        return arr

    def last_timing(self):
        a, b = ctypes.c_double(), ctypes.c_double()
        self._check(self.lib.igb_last_timing(self.h, ctypes.byref(a), ctypes.byref(b)), "igb_last_timing")
        return a.value, b.value

    def launch_count(self, reset=False):
        n = ctypes.c_longlong()
        self._check(self.lib.igb_launch_count(self.h, ctypes.byref(n), 1 if reset else 0), "igb_launch_count")
        return n.value

    def profile(self, on=True):
        self._check(self.lib.igb_profile_enable(self.h, 1 if on else 0), "igb_profile_enable")

    def profile_reset(self):
        self._check(self.lib.igb_profile_reset(self.h), "igb_profile_reset")

    def profile_get(self):
        out = {}
        for k, name in enumerate(KERNEL_CLASSES):
            ms, n, by = ctypes.c_double(), ctypes.c_longlong(), ctypes.c_double()
            self._check(self.lib.igb_profile_get(self.h, k, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(by)),
                        "igb_profile_get")
            fl = ctypes.c_double()
            self._check(self.lib.igb_profile_flops(self.h, k, ctypes.byref(fl)), "igb_profile_flops")
            tms, tn, tby = ctypes.c_double(), ctypes.c_longlong(), ctypes.c_double()
            self._check(self.lib.igb_profile_top(self.h, k, ctypes.byref(tms), ctypes.byref(tn), ctypes.byref(tby)),
                        "igb_profile_top")
            out[name] = {"ms": ms.value, "launches": n.value, "bytes": by.value, "flops": fl.value,
                         "top": {"ms": tms.value, "launches": tn.value, "bytes_per_launch": tby.value}}
        return out

    def gs_info(self, level, direction):
        """The Gauss-Seidel engine planned for (level, direction): dict with engine, B (flow: lanes
        per row), KA, KF, ranges (flow: CTAs), panels, depth, n."""
        info = (ctypes.c_int * 8)()
        self._check(self.lib.igb_gs_info(self.h, int(level), int(direction), info, 8), "igb_gs_info")
        v = list(info)
        return {"engine": GS_ENGINES.get(v[0], "?"), "B": v[1], "KA": v[2], "KF": v[3], "ranges": v[4],
                "panels": v[5], "depth": v[6], "n": v[7]}

    def cg(self, A, b, prec="none", prec_fn=None, tol=1e-8, max_iters=10000, callback=None):
        """igb_cg: PCG with any CSR operator (A None: the finest level's) and preconditioner
        ("none", "cycle": this context's cycle, "host": prec_fn(r) -> z on host arrays); callback(it,
        rel) is called after every iteration.  Returns (x, its, history)."""
        b = _c(b, np.float64)
        n = len(b)
        x = np.empty(n)
        hist = np.empty(max(1, int(max_iters)))
        its = ctypes.c_int(0)
        errors = []

        def _prec(r_ptr, z_ptr, nn, _user):
            try:
                r = np.ctypeslib.as_array(r_ptr, shape=(nn,))
                z = np.ctypeslib.as_array(z_ptr, shape=(nn,))
                z[:] = np.asarray(prec_fn(r.copy()), dtype=float)
            except BaseException as e:  # reported after the call (ctypes cannot propagate it)
                errors.append(e)

        def _iter(it, rel, _user):
            try:
                if callback is not None:
                    callback(int(it), float(rel))
            except BaseException as e:
                errors.append(e)

        pf = PREC_FN(_prec) if prec == "host" else PREC_FN()
        itf = ITER_FN(_iter) if callback is not None else ITER_FN()
        if A is None:
            args = (n, 0, None, None, None)
        else:
            import scipy.sparse
            A = scipy.sparse.csr_matrix(A)
            if not A.has_sorted_indices:
                A = A.sorted_indices()
            ip, ix, dv = _c(A.indptr, np.int32), _c(A.indices, np.int32), _c(A.data, np.float64)
            args = (n, A.nnz, _ptr(ip), _ptr(ix), _ptr(dv))
        rc = self.lib.igb_cg(self.h, *args, PREC[prec], ctypes.cast(pf, _p), None, ctypes.cast(itf, _p), None,
                             _ptr(b), float(tol), int(max_iters), _ptr(x), ctypes.byref(its), _ptr(hist), len(hist))
        if errors:
            raise errors[0]
        self._check(rc, "igb_cg")
        return x, its.value, hist[:its.value].tolist()

    def smooth(self, level, kind, post, steps, f, u):
        """igb_smooth: returns the iterate after `steps` pre- (post=False) or post-smoothing steps."""
        f = _c(f, np.float64)
        out = _c(u, np.float64).copy()
        self._check(self.lib.igb_smooth(self.h, int(level), SMOOTHER[kind], 1 if post else 0, int(steps),
                                        _ptr(f), _ptr(out)), "igb_smooth")
        return out

