"""Elliptic-mode orchestration on the GPU (reference `driver.py:20-146`).

`velocity_preconditioner` and `solve_elliptic` wire the drop-in pieces the
same way the reference's `solve_stokes(..., mode="elliptic")` does:
condense -> double Schur -> ASP(S_d) wrapped by ExtendedAsp -> PCG on the
condensed S.  The timings t_sup / t_sol follow `RunRecord` (`:33-57`), taken
with CUDA synchronisation so they are device times.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import preconditioners as pc
from .condensation import CondensedSystem, condense_sigma_omega, double_schur
from .dofmap import FeSystem
from .krylov import KrylovReport, cg
from .operators import SdOperator, SOperator


@dataclass
class SolverOptions:
    mode: str = "elliptic"
    target: str = "Sd"
    composition: str = "multiplicative"
    smoother: str = "jacobi"
    steps: int = 1
    penalty_C: float = 4.0
    rtol: float = 1e-6
    maxit: int = 500
    seed: int = 0


def build_system(problem, k, nu, opts: SolverOptions):
    fes = FeSystem(problem.mesh, problem.regions, k)
    sys_ = condense_sigma_omega(fes, nu, body_force=problem.body_force)
    if opts.target == "Sd":
        double_schur(sys_)
    return fes, sys_


def velocity_preconditioner(fes, sys_: CondensedSystem, nu, opts: SolverOptions):
    """ExtendedAsp(AspPreconditioner(S_d, facet Jacobi, E_c, coarse)) on the
    GPU (reference `driver.py:82-102`, target "Sd")."""
    if opts.target != "Sd":
        raise ValueError(f"GPU path supports target 'Sd' only, got {opts.target!r}")
    A = SdOperator(sys_)
    sm = pc.FacetBlockSmoother(A, None, opts.smoother)
    Ec = pc.embedding_cpl(fes, sys_)
    coarse = pc.build_coarse(fes, nu, penalty_C=opts.penalty_C)
    asp = pc.AspPreconditioner(A, sm, Ec, coarse, opts.composition, opts.steps)
    return pc.ExtendedAsp(sys_, asp)


def condensed_rhs(fes, sys_: CondensedSystem):
    """rhs_u = (load - S vv_values)[free] (reference `driver.py:105-110`);
    the Dirichlet lift is applied on the GPU when the data are nonzero."""
    load = sys_.load[fes.vv_free].copy()
    if np.any(fes.vv_values):
        # S @ vv_values over all dofs, restricted to free rows
        S = sys_.S
        load -= (S @ fes.vv_values)[fes.vv_free]
    return load


@dataclass
class EllipticResult:
    fes: FeSystem
    system: CondensedSystem
    x_free: object
    u: np.ndarray
    uhat: np.ndarray
    report: KrylovReport
    t_sup: float
    t_sol: float
    extras: dict = field(default_factory=dict)


def _sync():
    import torch
    torch.cuda.synchronize()


def solve_elliptic(problem, k, nu, opts: SolverOptions) -> EllipticResult:
    t0 = time.perf_counter()
    fes, sys_ = build_system(problem, k, nu, opts)
    M = velocity_preconditioner(fes, sys_, nu, opts)
    A = SOperator(sys_)
    rhs = condensed_rhs(fes, sys_)
    _sync()
    t_sup = time.perf_counter() - t0
    t1 = time.perf_counter()
    x, report = cg(A, rhs, M, rtol=opts.rtol, maxit=opts.maxit)
    _sync()
    t_sol = time.perf_counter() - t1
    x_full = fes.vv_values.copy()
    x_full[fes.vv_free] = x
    return EllipticResult(fes, sys_, x, x_full[:fes.n_v], x_full[fes.n_v:], report,
                          t_sup, t_sol)


def solve_stokes(problem, k, nu, opts: SolverOptions):
    if opts.mode != "elliptic":
        raise NotImplementedError(
            "Stokes (saddle/GMRES) mode is SURVEY §8f row 4; the GPU path covers "
            "the elliptic mode of the north star")
    return solve_elliptic(problem, k, nu, opts)
