"""The five BASELINE.json configurations, frozen as in SURVEY.md section 8(d).

Each builder returns a :class:`Problem` (hierarchy, cycle config, source
problem).  ``levels`` lets tests build the same configuration at fewer levels
(coarser finest grid) -- the coarse grid and everything else stay fixed.

  cfg1  unit square, p=2, 64^2 spans (coarse 8, L=3), SCMS smoother,
        f = 2 pi^2 sin(pi x) sin(pi y) (ManufacturedProblem(2))
  cfg2  [0,2]^2 as 2x2 unit patches, p=3, 128^2 spans/patch (coarse 4, L=5),
        hybrid, f = 2 pi^2 sin(pi x/2) sin(pi y/2), g = 0
  cfg3  L-shape, SIPG, non-matching 64/128/256 spans (coarse 4/8/16, L=4),
        p=4, hybrid, f = 1, g = 0, sigma = 5 (penalty with the global finest h)
  cfg4  [0,4]^2 as 4x4 bilinear patches perturbed by +-0.15 (seed 1),
        p in {2,4,6,8}, 256^2 spans/patch (coarse 4, L=6), hybrid,
        f = sin(pi x/2) sin(pi y/2), g = 0
  cfg5  [0,2]^3 as 2x2x2 unit cubes, p=3, 64^3 spans/patch (coarse 4, L=4),
        hybrid, ManufacturedProblem(3)
All: x0 = 0, tol = 1e-8, max_iters = 500, nu = mu = 1, tau = 1, delta = 0.12.
"""

from dataclasses import dataclass

import numpy as np

from . import assembly
from . import bspline as bs
from . import geometry as geom
from .multigrid import CycleConfig

__all__ = ["Problem", "build", "CONFIGS", "default_levels"]


@dataclass
class Problem:
    name: str
    hier: object
    config: CycleConfig
    problem: object

    def rhs(self, assembled):
        return assembly.assemble_rhs(self.hier, assembled, self.problem)


def _sin_half(scale):
    def f(X):
        X = np.asarray(X)
        return scale * np.prod(np.sin(0.5 * np.pi * X), axis=-1)
    return f


def _one(X):
    return np.ones(np.shape(X)[:-1])


def cfg1(levels=3):
    dom = geom.unit_square()
    hier = assembly.build_hierarchy(dom, 2, levels, "conforming", coarse_elements=8)
    return Problem("cfg1", hier, CycleConfig(smoother="scms", tau=1.0, delta=0.12),
                   assembly.ManufacturedProblem(2))


def cfg2(levels=5):
    dom = geom.square_grid(2, 2)
    hier = assembly.build_hierarchy(dom, 3, levels, coarse_elements=4)
    return Problem("cfg2", hier, CycleConfig(smoother="hyb"),
                   assembly.SourceProblem(_sin_half(2.0 * np.pi ** 2)))


def cfg3(levels=4):
    dom = geom.l_shape()
    p, coarse = 4, (4, 8, 16)
    spaces = [[(bs.open_knot_vector(p, c, lev),) * 2 for c in coarse] for lev in range(levels + 1)]
    hier = assembly.hierarchy_from_spaces(dom, p, levels, "dg", spaces, space_rule="nonmatching")
    return Problem("cfg3", hier, CycleConfig(smoother="hyb", tau=1.0, delta=0.12, sigma=5.0),
                   assembly.SourceProblem(_one))


def cfg4(p=2, levels=6):
    dom = geom.distorted_grid(4, 4, 0.15, seed=1)
    hier = assembly.build_hierarchy(dom, p, levels, coarse_elements=4)
    return Problem(f"cfg4_p{p}", hier, CycleConfig(smoother="hyb"),
                   assembly.SourceProblem(_sin_half(1.0)))


def cfg5(levels=4):
    dom = geom.box_grid((2, 2, 2))
    hier = assembly.build_hierarchy(dom, 3, levels, coarse_elements=4)
    return Problem("cfg5", hier, CycleConfig(smoother="hyb"), assembly.ManufacturedProblem(3))


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}


def default_levels(name):
    return {"cfg1": 3, "cfg2": 5, "cfg3": 4, "cfg4": 6, "cfg5": 4}[name]


def build(name, **kw):
    return CONFIGS[name](**kw)
