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
    """(rhs_u, rhs_p) with the Dirichlet lift (reference `driver.py:105-110`):
    rhs_u = (load - S vv_values)[free], rhs_p = -B vv_values.  The lift
    materialises S / B only when the Dirichlet data are nonzero (never for
    the BASELINE configs)."""
    load = sys_.load[fes.vv_free].copy()
    n_p = fes.dof_q.ndof
    if np.any(fes.vv_values):
        load -= (sys_.S @ fes.vv_values)[fes.vv_free]
        rhs_p = -(sys_.B @ fes.vv_values)
    else:
        rhs_p = np.zeros(n_p)
    return load, rhs_p


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
    rhs = condensed_rhs(fes, sys_)[0]
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


def pressure_projector(fes):
    """Remove the constant pressure mode from the trailing block of a stacked
    (velocity, pressure) device vector (reference `driver.py:113-130`)."""
    import torch
    from .operators import workspace
    loc = fes.dof_q.loc2glob
    one = np.zeros(fes.dof_q.ndof)
    one[loc[:, 0]] = 1.0 / fes.tab_q[0, 0]
    mass = np.zeros(fes.dof_q.ndof)
    mass[loc.ravel()] = (fes.detJ[:, None] * (fes.tab_q @ fes.quad_tri.weights)[None, :]).ravel()
    denom = float(mass @ one)
    nvfree = int(fes.vv_free.sum())
    one_d, mass_d = torch.from_numpy(one).cuda(), torch.from_numpy(mass).cuda()

    def project(x):
        out = x.clone()
        p = out[nvfree:]
        coef = workspace().dot_host(mass_d, p) / denom
        p.add_(one_d, alpha=-coef)
        return out

    project.mass, project.one = mass, one
    return project


@dataclass
class StokesResult:
    fes: FeSystem
    system: CondensedSystem
    x_free: object
    u: np.ndarray
    uhat: np.ndarray
    p: np.ndarray
    sigma: np.ndarray
    w: np.ndarray
    report: KrylovReport
    t_sup: float
    t_sol: float


def solve_stokes(problem, k, nu, opts: SolverOptions):
    """Reference `driver.py:133-180`: elliptic mode -> PCG on S; Stokes mode
    -> right-preconditioned GMRES on K = [[S, B^T], [B, 0]] with the block
    triangular saddle preconditioner (two ExtendedAsp applications, the
    diagonal pressure mass) and, for pure Dirichlet problems, the constant
    pressure mode projected out.  Both end with the GPU stress recovery."""
    if opts.mode == "elliptic":
        return solve_elliptic(problem, k, nu, opts)
    if opts.mode != "stokes":
        raise ValueError(f"unknown mode {opts.mode!r}")
    from .krylov import gmres
    from .operators import SaddleOperator
    t0 = time.perf_counter()
    fes, sys_ = build_system(problem, k, nu, opts)
    vel = velocity_preconditioner(fes, sys_, nu, opts)
    K = SaddleOperator(sys_)
    rhs_u, rhs_p = condensed_rhs(fes, sys_)
    mp = pc.PressureMassPrecond.build(fes, nu)
    saddle = pc.SaddlePreconditioner(vel, mp, K.B)
    mean_zero = bool(fes.regions.mean_zero_pressure)
    project = pressure_projector(fes) if mean_zero else None
    _sync()
    t_sup = time.perf_counter() - t0
    t1 = time.perf_counter()
    x, report = gmres(K, np.concatenate([rhs_u, rhs_p]), saddle, rtol=opts.rtol,
                      maxit=opts.maxit, project=project)
    _sync()
    t_sol = time.perf_counter() - t1
    nv = K.n_v
    x_free = x[:nv]
    p_phys = -x[nv:]
    if mean_zero:
        area = float(np.sum(fes.detJ) / 2.0)
        p_phys = p_phys - float(project.mass @ p_phys) / area * project.one
    x_full = fes.vv_values.copy()
    x_full[fes.vv_free] = x_free
    sigma, w = sys_.recover_stress(x_full)
    return StokesResult(fes, sys_, x_free, x_full[:fes.n_v], x_full[fes.n_v:], p_phys, sigma, w,
                        report, t_sup, t_sol)
