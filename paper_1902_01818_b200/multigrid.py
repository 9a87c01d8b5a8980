"""Multigrid driver: cycle configuration, solve reports and the device solver.

Drop-in for ``igamg.multigrid`` (``multigrid.py:20``): ``CycleConfig``,
``SolveReport`` and ``MultigridSolver`` with ``cycle``, ``preconditioner``,
``check_preconditioner_spd``, ``solve_pcg``, ``solve_stationary``,
``solve_direct`` and ``solve``.

Setup (finest assembly, prolongations, Galerkin coarse operators, coarse
factorization, smoother construction) runs on the host exactly as in the
reference (``multigrid.py:86-112``) and is timed separately
(``setup_seconds``).  Everything on the solve path -- the cycle and the whole
CG loop -- runs on one GPU through ``libigb`` (one upload per level; one
host<->device transfer of ``f``/``x`` per solve).
"""

import json
import os
import time
from dataclasses import dataclass, field, asdict

import numpy as np

from . import _setup_native
from . import assembly
from . import linsolve
from . import smoothers as sm
from ._lib import Context

__all__ = ["CycleConfig", "SolveReport", "MultigridSetup", "MultigridSolver", "DevicePreconditioner"]


@dataclass(frozen=True)
class CycleConfig:
    """Cycle / outer-iteration knobs (``multigrid.py:23-50``)."""

    smoother: str = "gs"
    mu: int = 1
    nu: int = 1
    nu_schedule: str = "constant"
    tau: float = 1.0
    delta: float = 0.12
    sigma: float = 5.0
    tol: float = 1e-8
    max_iters: int = 500
    interior_policy: str = "product"

    def __post_init__(self):
        if self.mu not in (1, 2):
            raise ValueError("cycle index mu must be 1 (V) or 2 (W)")
        if self.nu < 0 or self.tol <= 0:
            raise ValueError("invalid smoothing step count or tolerance")
        if self.smoother in ("scms", "hyb") and (self.tau <= 0 or self.delta <= 0):
            raise ValueError("scms/hybrid require positive damping and scaling")
        if self.smoother not in ("gs", "scms", "hyb"):
            raise ValueError(f"unknown smoother kind {self.smoother!r}")

    def steps_at(self, level, finest):
        if self.nu_schedule == "constant":
            return self.nu
        gap = finest - level
        return self.nu * 2 ** gap * (1 + gap) ** 2


@dataclass
class SolveReport:
    """Outcome of one solve (``multigrid.py:53-80``); ``x`` is the solution."""

    iterations: int
    converged: bool
    diverged: bool
    residuals: list
    wall_seconds: float
    n_dofs: int
    method: str
    config: dict
    x: np.ndarray = field(default=None, repr=False)
    device_ms: float = None

    @property
    def final_residual(self):
        return self.residuals[-1] if self.residuals else 0.0

    def to_json(self):
        return json.dumps({
            "iterations": self.iterations,
            "converged": self.converged,
            "diverged": self.diverged,
            "final_residual": self.final_residual,
            "wall_seconds": self.wall_seconds,
            "n_dofs": self.n_dofs,
            "method": self.method,
            "config": self.config,
        })


class DevicePreconditioner:
    """One cycle on the finest level from u = 0, as a linear operator on the device."""

    def __init__(self, solver):
        self.solver = solver

    def __call__(self, r):
        return self.solver.cycle(self.solver.finest, r)


class MultigridSetup:
    """Host-side setup of the hierarchy (``multigrid.py:86-112``), no device needed.

    Finest assembly, prolongations, Galerkin coarse operators ``P^T A P``,
    SuperLU coarse factorization and smoother construction; per-phase wall
    times in ``timings``.
    """

    def __init__(self, hier, config=CycleConfig(), assembled=None):
        t0 = time.perf_counter()
        self.hier = hier
        self.config = config
        self.finest = hier.L
        timings = {}
        t = time.perf_counter()
        asm = assembled if assembled is not None else assembly.assemble_level(hier, hier.L, sigma=config.sigma)
        timings["assemble"] = time.perf_counter() - t
        self.assembled_finest = asm
        self.A = [None] * (hier.L + 1)
        self.A[hier.L] = asm.A
        self.P = [None] * (hier.L + 1)
        t = time.perf_counter()
        for level in range(hier.L, 0, -1):
            self.P[level] = assembly.prolongation(hier, level)
            # Galerkin product (multigrid.py:95-99); native OpenMP product with SciPy's arithmetic
            # (csrc/host_setup.cpp, bit-identical), SciPy when the setup library is unavailable
            Ac = _setup_native.galerkin(self.A[level], self.P[level])
            if Ac is None:
                Ac = (self.P[level].T @ self.A[level] @ self.P[level]).tocsr()
            self.A[level - 1] = Ac
        timings["galerkin"] = time.perf_counter() - t
        t = time.perf_counter()
        self.coarse_solver = linsolve.factorize(self.A[0], spd=True)
        timings["coarse_factor"] = time.perf_counter() - t
        t = time.perf_counter()
        self.smoother = [None] * (hier.L + 1)
        for level in range(1, hier.L + 1):
            self.smoother[level] = sm.build_smoother(
                config.smoother, self.A[level], hier, level, tau=config.tau,
                delta=config.delta, interior_policy=config.interior_policy)
        timings["smoothers"] = time.perf_counter() - t
        self.timings = timings
        self.seconds = time.perf_counter() - t0

    @property
    def n_dofs(self):
        return self.A[self.finest].shape[0]

    def setup_bundle(self):
        """Plain setup data (matrices, transfers, piece/FD data) for independent checkers."""
        levels = [None]
        for level in range(1, self.finest + 1):
            smo = self.smoother[level]
            scms = smo if isinstance(smo, sm.SubspaceCorrectedMass) else getattr(smo, "scms", None)
            entry = {}
            if scms is not None:
                entry["tau"] = scms.tau
                entry["interiors"] = [
                    {"indices": p.indices, "dims": s.dims, "subspaces": s._subspaces}
                    for p, s in scms.interiors]
                entry["pieces"] = [p.indices for p, _ in scms.pieces]
            levels.append(entry)
        cfg = self.config
        return {
            "A": list(self.A), "P": list(self.P), "smoother": cfg.smoother, "mu": cfg.mu,
            "steps": [cfg.steps_at(l, self.finest) for l in range(self.finest + 1)],
            "levels": levels, "finest": self.finest,
        }


class MultigridSolver:
    """Assembled hierarchy + smoothers on the host, cycles and PCG on the GPU."""

    def __init__(self, hier, config=CycleConfig(), device=0, setup=None):
        t0 = time.perf_counter()
        self.setup = setup if setup is not None else MultigridSetup(hier, config)
        self.hier = hier
        self.config = config
        self.finest = hier.L
        self.assembled_finest = self.setup.assembled_finest
        self.A = self.setup.A
        self.P = self.setup.P
        self.coarse_solver = self.setup.coarse_solver
        self.smoother = self.setup.smoother
        t = time.perf_counter()
        self.ctx = Context(device)
        self._upload()
        self.setup_timings = dict(self.setup.timings, upload=time.perf_counter() - t)
        self.setup_seconds = self.setup.seconds + (time.perf_counter() - t0)
        self.coarse_calls = 0

    # -- upload ------------------------------------------------------------------
    def _upload(self):
        ctx, L, cfg = self.ctx, self.finest, self.config
        verbose = bool(os.environ.get("IGB_VERBOSE"))
        tick = [time.perf_counter()]

        def lap(what):
            if verbose:
                t = time.perf_counter()
                print(f"[igb] upload {what}: {t - tick[0]:.2f} s", flush=True)
                tick[0] = t

        ctx.set_num_levels(L)
        for level in range(L + 1):
            ctx.set_level_matrix(level, self.A[level])
        lap("level matrices")
        # matrix-free finest operator where the patches allow it and A_L is not tiny (measured: cfg2
        # 5.10 -> 5.04 ms; cfg1's 98K-nonzero level is launch-bound, 0.78 ms CSR vs 0.90 ms)
        # Coarser levels too: their Galerkin operators P^T A P equal the rediscretised ones the
        # sum factorisation applies to ~2e-15 relative (nested spaces, exact quadrature)
        min_nnz = int(os.environ.get("IGB_MATRIX_FREE_MIN_NNZ", 1_000_000))
        for level in range(1, L + 1):
            if self.A[level].nnz >= min_nnz:
                md = assembly.matrix_free_data(self.hier, level)
                if md is not None:
                    ctx.set_matrix_free(level, md)
        lap("matrix-free data")
        for level in range(1, L + 1):
            ctx.set_prolongation(level, self.P[level])
            if len(self.hier.spaces[level][0]) in (2, 3):
                ctx.set_prolongation_kron(level, assembly.prolongation_kron(self.hier, level))
        lap("prolongations")
        for level in range(1, L + 1):
            smo = self.smoother[level]
            gs = smo if isinstance(smo, sm.GaussSeidel) else getattr(smo, "gs", None)
            scms = smo if isinstance(smo, sm.SubspaceCorrectedMass) else getattr(smo, "scms", None)
            if scms is not None:
                ctx.scms_begin(level, scms.tau)
                for piece, solver in scms.interiors:
                    ctx.scms_add_interior(level, solver.dims, solver.square_transforms,
                                          solver.denominator, piece.indices)
                for i, ((piece, _), inv) in enumerate(zip(scms.pieces, scms.piece_inverses)):
                    if i in scms.tensor_faces:   # 3-D face with tensor structure: 2-D fast diagonalisation
                        fdims, fV, fden = scms.tensor_faces[i]
                        ctx.scms_add_interior(level, fdims, fV, fden, piece.indices)
                    else:
                        ctx.scms_add_piece(level, piece.indices, inv)
                lap(f"scms level {level}")
            if gs is not None:  # after the interiors (only the opt-in KF 10 panel variant reads the dimension)
                ctx.set_gs(level)
                lap(f"gs level {level}")
            smo.bind(ctx, level)
        Lf, Uf, pr, pc = self.coarse_solver.factors()
        ctx.set_coarse_lu(Lf, Uf, pr, pc)
        steps = [cfg.steps_at(level, L) for level in range(L + 1)]
        ctx.set_cycle(cfg.smoother, cfg.mu, steps)
        ctx.finalize()
        lap("coarse + finalize")

    @property
    def n_dofs(self):
        return self.A[self.finest].shape[0]

    def setup_bundle(self):
        return self.setup.setup_bundle()

    # -- solve-phase API -------------------------------------------------------------
    def cycle(self, level, f, u=None):
        """One cycle on ``level``; returns the new iterate (``multigrid.py:118-138``)."""
        if level < 1:
            raise ValueError("cycles act on levels >= 1")
        if level > self.finest:
            raise ValueError("level above the finest level")
        f = np.asarray(f, dtype=float)
        if u is None:
            return self.ctx.cycle(level, f)
        # cycle from u: residual-correction form u + B (f - A u), residual on the device
        res = self.ctx.op("residual", level, u, len(f), out_init=f)
        return u + self.ctx.cycle(level, res)

    def preconditioner(self):
        return DevicePreconditioner(self)

    def check_preconditioner_spd(self, rtol=1e-8, seed=20240801):
        """Symmetry/positivity of the cycle on a random pair (``multigrid.py:144-159``)."""
        rng = np.random.default_rng(seed)
        r = rng.standard_normal(self.n_dofs)
        s = rng.standard_normal(self.n_dofs)
        Br, Bs = self.cycle(self.finest, r), self.cycle(self.finest, s)
        lhs, rhs = s @ Br, r @ Bs
        scale = max(abs(lhs), abs(rhs), 1e-30)
        if abs(lhs - rhs) > rtol * scale:
            raise ValueError(
                "multigrid preconditioner is not symmetric "
                f"({abs(lhs - rhs) / scale:.2e} relative); use symmetric smoothing orders")
        if r @ Br <= 0 or s @ Bs <= 0:
            raise ValueError("multigrid preconditioner is not positive definite")

    def _report(self, its, converged, diverged, residuals, t0, method, x=None, device_ms=None):
        return SolveReport(its, converged, diverged, residuals, time.perf_counter() - t0,
                           self.n_dofs, method, asdict(self.config), x, device_ms)

    def solve_pcg(self, f, check_spd=True):
        """PCG with one cycle as preconditioner (``multigrid.py:236-251``); report carries x."""
        cfg = self.config
        t0 = time.perf_counter()
        f = np.asarray(f, dtype=float)
        if np.linalg.norm(f) == 0.0:
            return self._report(0, True, False, [], t0, "pcg", np.zeros_like(f))
        if check_spd:
            self.check_preconditioner_spd()
        x, its, history = self.ctx.pcg(f, cfg.tol, cfg.max_iters)
        converged = bool(history and history[-1] <= cfg.tol)
        return self._report(its, converged, not converged, history, t0, "pcg", x,
                            self.ctx.last_timing()[0])

    def _iterate(self, f, step, method):
        cfg = self.config
        t0 = time.perf_counter()
        normf = np.linalg.norm(f)
        if normf == 0.0:
            return self._report(0, True, False, [], t0, method, np.zeros_like(f))
        u = np.zeros_like(f)
        residuals = []
        increases = 0
        for it in range(1, cfg.max_iters + 1):
            u, rel = step(u)
            rel = rel / normf
            increases = increases + 1 if residuals and rel > residuals[-1] else 0
            residuals.append(rel)
            if rel <= cfg.tol:
                return self._report(it, True, False, residuals, t0, method, u)
            if increases >= 10 or not np.isfinite(rel):
                return self._report(it, False, True, residuals, t0, method, u)
        return self._report(cfg.max_iters, False, True, residuals, t0, method, u)

    def _residual(self, f, u):
        return self.ctx.op("residual", self.finest, u, len(f), out_init=f)

    def solve_stationary(self, f):
        """Repeated cycles from u = 0 (``multigrid.py:202-210``)."""
        f = np.asarray(f, dtype=float)

        def step(u):
            u = self.cycle(self.finest, f, u)
            return u, np.linalg.norm(self._residual(f, u))

        return self._iterate(f, step, "stationary")

    def solve_direct(self, f):
        """Cycle-preconditioned steepest descent with exact line search (``multigrid.py:212-234``)."""
        f = np.asarray(f, dtype=float)
        state = {"r": f.copy()}

        def step(u):
            r = state["r"]
            z = self.cycle(self.finest, r)
            Az = self.ctx.op("spmv", self.finest, z, len(z))
            zAz = z @ Az
            if not np.isfinite(zAz) or zAz <= 0.0:
                return u, np.inf
            alpha = (r @ z) / zAz
            u = u + alpha * z
            state["r"] = r - alpha * Az
            return u, np.linalg.norm(state["r"])

        return self._iterate(f, step, "direct")

    def solve(self, f, mode="direct"):
        if mode in ("direct", "d"):
            return self.solve_direct(f)
        if mode in ("pcg", "cg"):
            return self.solve_pcg(f)
        if mode in ("stationary", "richardson"):
            return self.solve_stationary(f)
        raise ValueError(f"unknown iteration mode {mode!r}")

    def close(self):
        self.ctx.close()
