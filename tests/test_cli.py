"""Command-line runner (paper_1902_01818_b200/cli.py; SPEC.md cli_runner): flag parsing, validation and
exit codes on the CPU, one device run per iteration mode on the GPU."""
import io
import contextlib

import pytest

from paper_1902_01818_b200 import cli


def _main(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = cli.main(argv)
    return rc, out.getvalue(), err.getvalue()


def test_flags_map_to_the_spec():
    a = cli.parser().parse_args("-g l_shape -r 5 -p 4 -s scms --MG.Damping .9 --MG.Scaling .12 --DG --NonMatching -i pcg".split())
    s = cli.spec_from_args(a)
    assert (s.geometry, s.refinements, s.degree, s.smoother) == ("l_shape", 5, 4, "scms")
    assert s.dg and s.nonmatching and s.iteration == "pcg" and s.damping == 0.9 and s.scaling == 0.12
    s.validate()


def test_validation_errors_exit_1():
    rc, out, err = _main("-g l_shape -r 3 -p 2 --NonMatching".split())
    assert rc == 1 and "requires --DG" in err
    rc, _, err = _main("-g l_shape -r 3 -p 2 -s scms --MG.Damping 0".split())
    assert rc == 1 and "positive" in err
    rc, _, err = _main("-g l_shape -r 3 -p 2 -s jacobi".split())
    assert rc == 1
    rc, _, err = _main("-g square_grid:2 -r 1 -p 2".split())
    assert rc == 1 and "malformed" in err


def test_builtin_geometries_resolve():
    assert cli.resolve_geometry("l_shape").num_patches == 3
    assert cli.resolve_geometry("square_grid:2x3").num_patches == 6
    assert cli.resolve_geometry("distorted:2x2:0.1:7").num_patches == 4
    assert cli.resolve_geometry("fichera").dim == 3


def test_missing_geometry_file_exits_3():
    rc, _, err = _main("-g /nonexistent/geometry.txt -r 1 -p 2".split())
    assert rc == 3 and "I/O error" in err


@pytest.mark.gpu
def test_runs_on_the_device_and_is_deterministic():
    rc, out, _ = _main("-g l_shape -r 3 -p 2 -s gs -i d --coarse-elements 2".split())
    rows = out.strip().splitlines()
    assert rc == 0 and rows[0] == cli.HEADER and len(rows) == 2
    its = int(rows[1].split(",")[5])
    assert 5 <= its <= 15                       # Table 1(a): 9 +- a few at these sizes
    rc2, out2, _ = _main("-g l_shape -r 3 -p 2 -s gs -i d --coarse-elements 2".split())
    assert out2.strip().splitlines()[1].split(",")[:7] == rows[1].split(",")[:7]   # identical counts and residual
    rc, out, _ = _main("-g square_grid:2x2 -r 3 -p 3 -s hyb -i pcg --coarse-elements 2 --table 2:3 2:3".split())
    assert rc == 0 and len(out.strip().splitlines()) == 5
