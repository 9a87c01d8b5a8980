"""Outputs and formats around the solve path: COO dumps (linsolve.py:113-131), the
plain-text geometry format (geometry.py:474-540), solution_coefficients / l2_error
(assembly.py:726-755), dense_generalized_eig (linsolve.py:104-110).  Host code, CPU tests; against
the reference itself when it is importable here."""

import os
import sys

import numpy as np
import pytest
import scipy.linalg
import scipy.sparse
import scipy.sparse.linalg

from conftest import REFERENCE_SRC, get_setup

HAVE_REF = os.path.isdir(REFERENCE_SRC)


def _ref():
    sys.path.insert(0, REFERENCE_SRC)
    import igamg.assembly as ra
    import igamg.geometry as rg
    import igamg.linsolve as rl
    return ra, rg, rl


def test_coo_round_trip_exact(tmp_path):
    from paper_1902_01818_b200 import linsolve
    pr, setup, f = get_setup("cfg2", levels=2)
    A = setup.A[1]
    linsolve.write_coo(tmp_path / "a.coo", A)
    B = linsolve.read_coo(tmp_path / "a.coo")
    assert B.shape == A.shape and (B != A).nnz == 0
    if HAVE_REF:
        ra, rg, rl = _ref()
        rl.write_coo(tmp_path / "r.coo", A)
        assert (tmp_path / "a.coo").read_text() == (tmp_path / "r.coo").read_text()
        assert (rl.read_coo(tmp_path / "a.coo") != A).nnz == 0


def test_geometry_text_round_trip(tmp_path):
    from paper_1902_01818_b200 import geometry
    dom = geometry.distorted_grid(2, 3, 0.1, seed=5)
    geometry.write_geometry(tmp_path / "g.txt", dom)
    back = geometry.read_geometry(tmp_path / "g.txt")
    assert back.num_patches == dom.num_patches and len(back.interfaces) == len(dom.interfaces)
    for p, q in zip(dom.patches, back.patches):
        assert p.spaces == q.spaces and np.array_equal(p.control_points, q.control_points)
    X0, J0 = geometry.eval_map(dom.patches[1], np.array([0.3, 0.6]))
    X1, J1 = geometry.eval_map(back.patches[1], np.array([0.3, 0.6]))
    assert np.array_equal(X0, X1) and np.array_equal(J0, J1)
    if HAVE_REF:
        ra, rg, rl = _ref()
        rg.write_geometry(tmp_path / "r.txt", rg.distorted_grid(2, 3, 0.1, seed=5))
        assert (tmp_path / "g.txt").read_text() == (tmp_path / "r.txt").read_text()
        rb = rg.read_geometry(tmp_path / "g.txt")
        assert rb.num_patches == back.num_patches and len(rb.interfaces) == len(back.interfaces)


def test_bad_geometry_file_is_an_error(tmp_path):
    from paper_1902_01818_b200 import geometry
    (tmp_path / "x.txt").write_text("not a geometry\n")
    with pytest.raises(geometry.GeometryError):
        geometry.read_geometry(tmp_path / "x.txt")


def test_side_point_on_the_boundary():
    from paper_1902_01818_b200 import geometry
    dom = geometry.unit_square()
    side = geometry.Side(0, 1)
    assert np.allclose(geometry.side_point(dom.patches[0], side, 0.25), [1.0, 0.25])


def test_l2_error_matches_reference_and_converges():
    from paper_1902_01818_b200 import assembly, configs, multigrid
    errs = []
    for levels in (1, 2):
        pr = configs.build("cfg1", levels=levels)
        setup = multigrid.MultigridSetup(pr.hier, pr.config)
        asm = setup.assembled_finest
        u = scipy.sparse.linalg.spsolve(setup.A[setup.finest].tocsc(), pr.rhs(asm))
        errs.append(assembly.l2_error(pr.hier, asm, u, pr.problem))
    assert errs[1] < errs[0] / 6  # p = 2: O(h^3) in L2
    if HAVE_REF:
        ra, rg, rl = _ref()
        rh = ra.build_hierarchy(rg.unit_square(), 2, 2, "conforming", coarse_elements=8)
        rasm = ra.assemble_level(rh, 2)
        rf = ra.assemble_rhs(rh, rasm, ra.ManufacturedProblem(2))
        ru = scipy.sparse.linalg.spsolve(rasm.A.tocsc(), rf)
        ref = ra.l2_error(rh, rasm, ru, ra.ManufacturedProblem(2))
        assert abs(errs[1] - ref) <= 1e-9 * ref


def test_dense_generalized_eig():
    from paper_1902_01818_b200 import linsolve
    rng = np.random.default_rng(2)
    Q = rng.standard_normal((6, 6))
    A = Q + Q.T
    B = Q @ Q.T + 6 * np.eye(6)
    lam = linsolve.dense_generalized_eig(scipy.sparse.csr_matrix(A), B)
    assert np.allclose(lam, scipy.linalg.eigh(A, B, eigvals_only=True))
    with pytest.raises(ValueError):
        linsolve.dense_generalized_eig(A, np.eye(5))


def test_coercivity_and_geometry_diagnostics():
    from paper_1902_01818_b200 import assembly
    pr, setup, f = get_setup("cfg3", levels=1)
    asm = setup.assembled_finest
    lam = assembly.check_coercivity(asm)
    assert lam > 0
    lo, hi, ratio = assembly.geometry_condition_diagnostic(setup.A[0], setup.A[0])
    assert abs(lo - 1) < 1e-10 and abs(hi - 1) < 1e-10 and abs(ratio - 1) < 1e-10
