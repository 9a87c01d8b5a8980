"""Command-line experiment runner (SPEC.md `cli_runner`; the reference declares `igamg.cli:main` in
pkg/pyproject.toml:19 but ships no module).  Flags mirror the paper's listings:

  python -m paper_1902_01818_b200.cli -g l_shape -r 4 -p 2 -s gs -i d
  python -m paper_1902_01818_b200.cli -g l_shape -r 5 -p 4 -s scms --MG.Damping .9 --MG.Scaling .12 \
        --DG --NonMatching -i pcg
  python -m paper_1902_01818_b200.cli -g fichera -r 3 -p 3 -s hyb -i pcg --table 2:3 2:3

Geometries: l_shape, fichera, unit_square, square_grid:RxC, box_grid:AxBxC, distorted:RxC:amp:seed, or a
geometry file (geometry.read_geometry).  Output: one CSV row per run -- domain, mode, smoother, p, L,
iterations, final relative residual, wall seconds -- on standard output or --out FILE.  Exit status: 0
converged, 1 validation error, 2 divergence / iteration cap, 3 I/O error.  The solve runs on the device
(MultigridSolver); there is no CPU fallback.
"""
import argparse
import sys
import time
from dataclasses import dataclass

import numpy as np

HEADER = "domain,mode,smoother,p,L,iterations,final_rel_residual,wall_seconds"


@dataclass
class ExperimentSpec:
    geometry: str
    refinements: int
    degree: int
    smoother: str = "gs"
    dg: bool = False
    nonmatching: bool = False
    damping: float = 1.0
    scaling: float = 0.12
    penalty: float = 5.0
    iteration: str = "direct"
    cycle: int = 1
    smoothing_steps: int = 1
    coarse_elements: int = 1
    tol: float = 1e-8
    max_iters: int = 500

    def validate(self):
        if self.nonmatching and not self.dg:
            raise ValueError("--NonMatching requires --DG")
        if self.smoother not in ("gs", "scms", "hyb"):
            raise ValueError(f"unknown smoother {self.smoother!r}")
        if self.smoother in ("scms", "hyb") and not (self.damping > 0 and self.scaling > 0):
            raise ValueError("scms / hyb need positive --MG.Damping and --MG.Scaling")
        if self.iteration not in ("direct", "pcg"):
            raise ValueError(f"unknown iteration mode {self.iteration!r}")
        if self.refinements < 1 or self.degree < 1:
            raise ValueError("need -r >= 1 and -p >= 1")
        if self.cycle not in (1, 2):
            raise ValueError("--cycle must be 1 (V) or 2 (W)")


def resolve_geometry(name):
    """Builtin name or geometry file -> MultiPatchDomain (ValueError for a bad name, OSError for a bad file)."""
    from . import geometry as geom
    head, *args = name.split(":")
    builtin = ("l_shape", "fichera", "unit_square", "square_grid", "box_grid", "distorted")
    if head in builtin:
        try:
            return _builtin_geometry(geom, head, args)
        except (ValueError, TypeError):
            raise ValueError(f"malformed geometry {name!r}") from None
    return geom.read_geometry(name)


def _builtin_geometry(geom, head, args):
    if head == "l_shape" and not args:
        return geom.l_shape()
    if head == "fichera" and not args:
        return geom.fichera()
    if head == "unit_square" and not args:
        return geom.unit_square()
    if head == "square_grid" and len(args) == 1:
        r, c = (int(v) for v in args[0].split("x"))
        return geom.square_grid(r, c)
    if head == "box_grid" and len(args) == 1:
        return geom.box_grid(tuple(int(v) for v in args[0].split("x")))
    if head == "distorted" and len(args) == 3:
        r, c = (int(v) for v in args[0].split("x"))
        return geom.distorted_grid(r, c, float(args[1]), seed=int(args[2]))
    raise ValueError("malformed")


def _unit_source(X):
    return np.ones(np.shape(X)[:-1])


def run(spec, device=0):
    """One experiment -> (SolveReport, CSV row)."""
    from . import assembly, multigrid
    spec.validate()
    dom = resolve_geometry(spec.geometry)
    mode = "dg" if spec.dg else "conforming"
    rule = "nonmatching" if spec.nonmatching else "matching"
    hier = assembly.build_hierarchy(dom, spec.degree, spec.refinements, mode, rule, spec.coarse_elements)
    cfg = multigrid.CycleConfig(smoother=spec.smoother, mu=spec.cycle, nu=spec.smoothing_steps, tau=spec.damping,
                                delta=spec.scaling, sigma=spec.penalty, tol=spec.tol, max_iters=spec.max_iters)
    t = time.perf_counter()
    solver = multigrid.MultigridSolver(hier, cfg, device=device)
    try:
        f = assembly.assemble_rhs(hier, solver.assembled_finest, assembly.SourceProblem(_unit_source))
        rep = solver.solve(f, mode=spec.iteration)
    finally:
        solver.close()
    wall = time.perf_counter() - t
    final = rep.residuals[-1] if len(rep.residuals) else 0.0
    row = (f"{spec.geometry},{mode}{'+nonmatching' if spec.nonmatching else ''}:{spec.iteration},{spec.smoother},"
           f"{spec.degree},{spec.refinements},{rep.iterations},{final:.6e},{wall:.3f}")
    return rep, row


def _range(text):
    lo, _, hi = text.partition(":")
    return range(int(lo), int(hi or lo) + 1)


def parser():
    ap = argparse.ArgumentParser(prog="igamg", description="Multigrid experiments for multi-patch IgA (device solve)")
    ap.add_argument("-g", "--geometry", required=True)
    ap.add_argument("-r", "--refinements", type=int, required=True)
    ap.add_argument("-p", "--degree", type=int, required=True)
    ap.add_argument("-s", "--smoother", default="gs")
    ap.add_argument("-i", "--iteration", default="d", help="d (direct / stationary V-cycle iteration) or pcg")
    ap.add_argument("--DG", dest="dg", action="store_true")
    ap.add_argument("--NonMatching", dest="nonmatching", action="store_true")
    ap.add_argument("--MG.Damping", dest="damping", type=float, default=1.0)
    ap.add_argument("--MG.Scaling", dest="scaling", type=float, default=0.12)
    ap.add_argument("--penalty", type=float, default=5.0)
    ap.add_argument("--cycle", type=int, default=1)
    ap.add_argument("--smoothing-steps", type=int, default=1)
    ap.add_argument("--coarse-elements", type=int, default=1)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--max-iters", type=int, default=500)
    ap.add_argument("--table", nargs=2, metavar=("L_RANGE", "P_RANGE"),
                    help="run every (L, p) of lo:hi ranges instead of the single (-r, -p) cell")
    ap.add_argument("--out", help="CSV file (default: standard output)")
    ap.add_argument("--device", type=int, default=0)
    return ap


def spec_from_args(a, L=None, p=None):
    it = {"d": "direct", "direct": "direct", "pcg": "pcg", "cg": "pcg"}.get(a.iteration, a.iteration)
    return ExperimentSpec(a.geometry, a.refinements if L is None else L, a.degree if p is None else p, a.smoother,
                          a.dg, a.nonmatching, a.damping, a.scaling, a.penalty, it, a.cycle, a.smoothing_steps,
                          a.coarse_elements, a.tol, a.max_iters)


def main(argv=None):
    a = parser().parse_args(argv)
    cells = [(None, None)]
    if a.table:
        cells = [(L, p) for L in _range(a.table[0]) for p in _range(a.table[1])]
    try:
        for L, p in cells:
            spec_from_args(a, L, p).validate()
    except ValueError as e:
        print(f"validation error: {e}", file=sys.stderr)
        return 1
    try:
        out = open(a.out, "w") if a.out else sys.stdout
    except OSError as e:
        print(f"I/O error: {e}", file=sys.stderr)
        return 3
    status = 0
    print(HEADER, file=out)
    for L, p in cells:   # deterministic (L, p) order; a cell's error is recorded in its row
        spec = spec_from_args(a, L, p)
        try:
            rep, row = run(spec, a.device)
            if not rep.converged:
                status = max(status, 2)
        except OSError as e:
            print(f"I/O error: {e}", file=sys.stderr)
            return 3
        except ValueError as e:
            if not a.table:
                print(f"validation error: {e}", file=sys.stderr)
                return 1
            row = f"{spec.geometry},error,{spec.smoother},{spec.degree},{spec.refinements},,{e},"
            status = max(status, 1)
        print(row, file=out, flush=True)
    if a.out:
        out.close()
    return status


if __name__ == "__main__":
    sys.exit(main())
