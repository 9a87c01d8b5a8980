"""Wave-sweep planner (csrc/wave_plan.cpp) on the CPU: the plan is emulated frame by frame on the
host (tests/native/wave_plan_emul.cpp) and must be a valid schedule that reproduces the
substitution of the reference's Gauss-Seidel sweeps (smoothers.py:178-190) on tril(A) / triu(A)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1902_01818_b200", "csrc")


@pytest.fixture(scope="module")
def emul(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("wave") / "libwave_emul.so")
    subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", "-I" + CSRC, "-o", out,
                    os.path.join(ROOT, "tests", "native", "wave_plan_emul.cpp"), os.path.join(CSRC, "wave_plan.cpp")],
                   check=True)
    lib = ctypes.CDLL(out)
    lib.wave_plan_emulate.restype = ctypes.c_int
    return lib


def band(n, p, rng):
    """SPD-like banded 1-D matrix of half bandwidth p."""
    a = sp.diags([rng.uniform(0.1, 1.0, n - abs(k)) for k in range(-p, p + 1)], range(-p, p + 1), format="csr")
    return (a + a.T + 4 * (p + 1) * sp.identity(n)).tocsr()


def kron3(a, b, c):
    A = sp.kron(sp.kron(a, b, format="csr"), c, format="csr")
    A.eliminate_zeros()   # sp.kron builds dense blocks with explicit zeros
    return A


def run(lib, A, upper, rb_min=32, rb_cap=8192, groups=148, late_lag=9, ewarps=7):
    A = A.tocsr()
    A.sort_indices()
    n = A.shape[0]
    ptr = A.indptr.astype(np.int32)
    col = A.indices.astype(np.int32)
    val = A.data.astype(np.float64)
    dpos = np.array([ptr[i] + np.searchsorted(col[ptr[i]:ptr[i + 1]], i) for i in range(n)], dtype=np.int32)
    rhs = np.random.default_rng(3).standard_normal(n)
    x = np.zeros(n)
    stats = np.zeros(16, dtype=np.int32)
    P = ctypes.POINTER
    rc = lib.wave_plan_emulate(n, ptr.ctypes.data_as(P(ctypes.c_int)), col.ctypes.data_as(P(ctypes.c_int)),
                               val.ctypes.data_as(P(ctypes.c_double)), dpos.ctypes.data_as(P(ctypes.c_int)),
                               int(upper), rb_min, rb_cap, late_lag, groups, ewarps, rhs.ctypes.data_as(P(ctypes.c_double)),
                               x.ctypes.data_as(P(ctypes.c_double)), stats.ctypes.data_as(P(ctypes.c_int)))
    T = sp.triu(A, format="csr") if upper else sp.tril(A, format="csr")
    ref = spsolve_triangular(T, rhs, lower=not upper)
    return rc, x, ref, stats


@pytest.mark.parametrize("upper", [False, True])
def test_3d_lexicographic_planes_are_bundles(emul, upper):
    rng = np.random.default_rng(0)
    n0, n1, n2, p = 6, 9, 11, 3
    A = kron3(band(n0, p, rng), band(n1, p, rng), band(n2, p, rng))
    rc, x, ref, st = run(emul, A, upper)
    assert rc == 0, rc
    assert np.linalg.norm(x - ref) <= 1e-13 * np.linalg.norm(ref)
    assert st[0] == n0 and st[3] == n1 * n2          # one bundle per plane
    assert st[5] == 0                                 # p = 3: the 24 in-plane neighbours all stay internal
    assert st[7] == (n2 - 1) + (p + 1) * (n1 - 1) + (p + 1) ** 2 * (n0 - 1) + 1   # depth of the lattice
    assert st[8] == A.shape[0]


@pytest.mark.parametrize("upper", [False, True])
def test_two_patches_sharing_a_face_and_random_couplings(emul, upper):
    rng = np.random.default_rng(1)
    blk = kron3(band(5, 3, rng), band(6, 3, rng), band(7, 3, rng))
    n = blk.shape[0]
    C = sp.random(n, n, density=2e-3, random_state=5, format="csr")
    A = sp.bmat([[blk, C], [C.T, blk]], format="csr")
    for ewarps, groups in ((1, 148), (5, 148), (64, 20)):
        rc, x, ref, st = run(emul, A, upper, ewarps=ewarps, groups=groups)
        assert rc == 0, (rc, ewarps, groups)
        assert np.linalg.norm(x - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("upper", [False, True])
def test_2d_high_degree_demotes_old_internal_entries(emul, upper):
    rng = np.random.default_rng(2)
    A = sp.kron(band(20, 5, rng), band(40, 5, rng), format="csr")
    A.eliminate_zeros()
    rc, x, ref, st = run(emul, A, upper, rb_cap=256)
    assert rc == 0, rc
    assert st[5] > 0                                  # more than 24 in-bundle entries per row
    assert np.linalg.norm(x - ref) <= 1e-13 * np.linalg.norm(ref)


def test_occupancy_bound_rejects_too_few_groups(emul):
    rng = np.random.default_rng(0)
    A = kron3(band(12, 3, rng), band(9, 3, rng), band(9, 3, rng))
    rc, _, _, st = run(emul, A, False, groups=2)
    assert rc == 1 and st[1] > 2
    rc, _, _, st = run(emul, A, False, groups=16)
    assert rc == 0 and st[1] <= 16
