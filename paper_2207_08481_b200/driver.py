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
from typing import Optional

import numpy as np

from . import preconditioners as pc
from .condensation import CondensedSystem, condense_sigma_omega, double_schur
from .dofmap import FeSystem
from .krylov import KrylovReport, cg
from .operators import SdOperator, SOperator


@dataclass
class SolverOptions:
    """Reference `driver.py:20-30`, same defaults.  The GPU preconditioner
    implements smoother "jacobi" (the north-star target); "gauss_seidel"
    (the reference default) and "l1" raise NotImplementedError when a
    preconditioner is actually built with them."""
    mode: str = "stokes"               # stokes | elliptic
    target: str = "Sd"                 # S | Sd (preconditioner target)
    composition: str = "multiplicative"
    smoother: str = "gauss_seidel"     # gauss_seidel | jacobi | l1
    steps: int = 1
    penalty_C: float = 4.0
    rtol: float = 1e-6
    maxit: int = 500
    seed: int = 0


@dataclass
class RunRecord:
    """Reference `driver.py:33-57` (timings are device-synchronised)."""
    problem: str
    k: int
    level: int
    n_elements: int
    n_dofs: int                 # free dofs of (V x Vhat) x Q
    iterations: int
    t_tot: float
    t_sup: float
    t_sol: float
    converged: bool
    max_div: float = np.nan
    nt_jump: float = np.nan
    lambda_min: Optional[float] = None
    lambda_max: Optional[float] = None
    cond: Optional[float] = None

    CSV_FIELDS = ["problem", "k", "level", "n_elements", "n_dofs",
                  "iterations", "t_tot", "t_sup", "t_sol", "converged",
                  "max_div", "nt_jump", "lambda_min", "lambda_max", "cond"]

    def csv_row(self):
        vals = [getattr(self, f) for f in self.CSV_FIELDS]
        return [("" if v is None else v) for v in vals]


def build_system(problem, k, nu, opts: SolverOptions):
    fes = FeSystem(problem.mesh, problem.regions, k)
    sys_ = condense_sigma_omega(fes, nu, body_force=problem.body_force)
    if opts.target == "Sd":
        double_schur(sys_)
    return fes, sys_


def velocity_preconditioner(fes, sys_: CondensedSystem, nu, opts: SolverOptions):
    """ExtendedAsp(AspPreconditioner(S_d, facet Jacobi, E_c, coarse)) on the
    GPU (reference `driver.py:82-102`, target "Sd")."""
    if opts.target == "S":
        raise NotImplementedError(
            "preconditioner target 'S' (overlapping facet_blocks_full) is outside the GPU "
            "scope (SURVEY §2); use target='Sd'")
    if opts.target != "Sd":
        raise ValueError(f"unknown preconditioner target {opts.target!r}")
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
class SolveResult:
    """Reference `driver.py:60-71`; `p` is None in elliptic mode.  `x_free`
    (the Krylov solution on free dofs) is an addition."""
    fes: FeSystem
    system: CondensedSystem
    u: np.ndarray               # V coefficients, Dirichlet data included
    uhat: np.ndarray
    p: Optional[np.ndarray]     # physical pressure
    sigma: np.ndarray
    w: np.ndarray
    report: KrylovReport
    record: RunRecord
    checks: dict = field(default_factory=dict)
    x_free: object = None

    @property
    def t_sup(self):
        return self.record.t_sup

    @property
    def t_sol(self):
        return self.record.t_sol


# earlier names of the two result kinds
EllipticResult = StokesResult = SolveResult


def _record(problem, fes, k, report, t0, t_sup, t_sol, checks):
    """RunRecord exactly as `driver.py:170-177` fills it."""
    return RunRecord(problem=getattr(problem, "name", ""), k=k, level=-1,
                     n_elements=fes.mesh.num_triangles,
                     n_dofs=int(fes.vv_free.sum()) + fes.dof_q.ndof,
                     iterations=report.iterations,
                     t_tot=time.perf_counter() - t0, t_sup=t_sup, t_sol=t_sol,
                     converged=report.converged,
                     max_div=checks["max_div_scaled"], nt_jump=checks["nt_jump_scaled"])


def _sync():
    import torch
    torch.cuda.synchronize()


def solve_elliptic(problem, k, nu, opts: SolverOptions) -> SolveResult:
    """Elliptic branch of `driver.solve_stokes` (`driver.py:143-146`)."""
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
    # reference driver.py:164-177: stress recovery, structural checks, record
    sigma, w = sys_.recover_stress(x_full)
    checks = post_checks(fes, sys_, x_full[:fes.n_v], sigma, report)
    record = _record(problem, fes, k, report, t0, t_sup, t_sol, checks)
    return SolveResult(fes=fes, system=sys_, u=x_full[:fes.n_v], uhat=x_full[fes.n_v:], p=None,
                       sigma=sigma, w=w, report=report, record=record, checks=checks, x_free=x)


def post_checks(fes, sys_, u, sigma, report: KrylovReport) -> dict:
    """Structural postconditions (reference `driver.py:183-218`): pointwise
    divergence scaled by the H1 seminorm, nt-continuity of the recovered
    stress across interior facets, residual monotonicity.  The element and
    facet sweeps run on the GPU (csrc/postcheck.cu)."""
    import torch
    from . import _abi
    dev = lambda a, dt=np.float64: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).cuda()
    nt = fes.mesh.num_triangles
    nu_l = fes.tab_u_div.shape[0]
    nq = fes.tab_u_div.shape[1]
    geo = np.zeros((nt, 10))
    geo[:, 0:4] = fes.J.reshape(nt, 4)
    geo[:, 4:8] = fes.Jinv.reshape(nt, 4)
    geo[:, 8] = fes.detJ
    dv = fes.dof_v
    vcodes = (2 * dv.loc2glob + (dv.signs < 0)).astype(np.int32)
    mesh = fes.mesh
    fint = np.asarray(mesh.interior_facets)
    t01 = mesh.facet_tri[fint]
    le = np.stack([np.argmax(fes.edge_facet[t01[:, s_]] == fint[:, None], axis=1) for s_ in (0, 1)], 1)
    fac = np.stack([t01[:, 0], le[:, 0], t01[:, 1], le[:, 1]], 1).astype(np.int32)
    frame = np.concatenate([mesh.facet_tangent[fint], mesh.facet_normal[fint]], 1)
    ns = fes.tab_sigma_edge.shape[0]
    nqe = fes.tab_sigma_edge.shape[2]
    nparts = 4 * 148 * 4
    out = torch.zeros(4, dtype=torch.float64, device="cuda")
    part = torch.zeros(nparts, dtype=torch.float64, device="cuda")
    u_d, s_d = dev(u), dev(sigma)
    args = [dev(geo), dev(vcodes, np.int32), u_d, dev(fes.tab_u_div), dev(fes.tab_u_grad),
            dev(fes.quad_tri.weights), len(fint), ns, nqe, dev(fac, np.int32), dev(frame),
            dev(fes.edge_flip.astype(np.int8), np.int8), s_d, dev(fes.tab_sigma_edge)]
    ptrs = [a if isinstance(a, int) else _abi.ptr(a) for a in args]
    _abi.call("mcs_post_checks", nt, nu_l, nq, *ptrs, _abi.ptr(out), _abi.ptr(part), nparts,
              _abi.stream(None))
    o = out.cpu().numpy()
    grad_scale = max(1.0, float(np.sqrt(np.sum(part.cpu().numpy()))))
    res = report.residuals
    monotone = all(res[i + 1] <= res[i] * (1 + 1e-12) for i in range(len(res) - 1))
    return {"max_div_scaled": float(o[0]) / grad_scale,
            "nt_jump_scaled": float(o[1]) / max(float(o[2]), 1.0),
            "residual_monotone": monotone}


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


def solve_stokes(problem, k, nu, opts: SolverOptions) -> SolveResult:
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
    checks = post_checks(fes, sys_, x_full[:fes.n_v], sigma, report)
    record = _record(problem, fes, k, report, t0, t_sup, t_sol, checks)
    return SolveResult(fes=fes, system=sys_, u=x_full[:fes.n_v], uhat=x_full[fes.n_v:],
                       p=p_phys, sigma=sigma, w=w, report=report, record=record,
                       checks=checks, x_free=x_free)
