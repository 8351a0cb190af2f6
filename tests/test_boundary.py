"""The drop-in boundary of SURVEY §8(b): the reference's CondensedSystem
attribute/method surface, SolverOptions / SolveResult, and the preconditioner
pieces built from reference-typed inputs (SciPy CSR + block lists, the
reference's CoarseSolver, NumPy callables in cg), all against the golden
fixtures the reference itself produced (oracle/make_golden.py).

Reference tests mirrored: test_condensation.py:77-83 (harmonic extension
idempotent / contractive), :123-143 (apply_S_factorized vs S @ x, incl.
bubble-only input), test_preconditioners.py:225-229 (Jacobi on the blocks)."""
import dataclasses
import inspect
import os

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden, rel
from paper_2207_08481_b200 import driver as D
from paper_2207_08481_b200 import preconditioners as pc
from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur
from paper_2207_08481_b200.dofmap import FeSystem
from paper_2207_08481_b200.problems import baseline_config

REF_SRC = "/root/reference/pkg/src"
CASES = ["c1_n2", "c2_n3", "c3_n2"]


def _csr(g, p):
    return sp.csr_matrix((g[p + "_data"], g[p + "_indices"], g[p + "_indptr"]),
                         shape=tuple(g[p + "_shape"]))


def _system(g):
    prob = baseline_config(int(g["cfg"]), int(g["n"]))
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    return prob, fes, double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))


# ------------------------------------------------------------------ CPU


def test_solver_options_defaults_are_the_reference_defaults():
    """driver.py:20-30."""
    o = D.SolverOptions()
    assert (o.mode, o.target, o.composition, o.smoother, o.steps, o.penalty_C, o.rtol,
            o.maxit, o.seed) == ("stokes", "Sd", "multiplicative", "gauss_seidel", 1, 4.0,
                                 1e-6, 500, 0)


def test_result_types_have_the_reference_fields():
    """driver.py:33-71: RunRecord (incl. CSV_FIELDS / csv_row) and SolveResult."""
    want = ["fes", "system", "u", "uhat", "p", "sigma", "w", "report", "record", "checks"]
    assert [f.name for f in dataclasses.fields(D.SolveResult)][:len(want)] == want
    assert D.RunRecord.CSV_FIELDS == ["problem", "k", "level", "n_elements", "n_dofs",
                                      "iterations", "t_tot", "t_sup", "t_sol", "converged",
                                      "max_div", "nt_jump", "lambda_min", "lambda_max", "cond"]
    r = D.RunRecord("p", 2, -1, 8, 10, 3, 1.0, 0.5, 0.5, True)
    assert r.csv_row()[-3:] == ["", "", ""]


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present (GPU box)")
def test_entry_point_signatures_match_the_reference():
    """Every §8(b) entry point takes the reference's parameters (names, order,
    defaults); additions are keyword-only extras at the end (stream, E=None)."""
    import importlib
    import sys
    sys.path.insert(0, REF_SRC)
    try:
        ref = {m: importlib.import_module(f"mcstokes.{m}") for m in
               ("condensation", "preconditioners", "driver", "krylov")}
    finally:
        sys.path.remove(REF_SRC)
    from paper_2207_08481_b200 import condensation, krylov
    ours = dict(condensation=condensation, preconditioners=pc, driver=D, krylov=krylov)
    names = {
        "condensation": ["condense_sigma_omega", "double_schur"],
        "preconditioners": ["build_embedding", "embedding_cpl", "build_coarse",
                            "facet_blocks_schur", "FacetBlockSmoother", "AspPreconditioner",
                            "ExtendedAsp", "PressureMassPrecond", "SaddlePreconditioner"],
        "driver": ["velocity_preconditioner", "condensed_rhs", "solve_stokes", "build_system",
                   "post_checks", "pressure_projector"],
        "krylov": ["cg", "gmres"],
    }
    for mod, fns in names.items():
        for fn in fns:
            rs = inspect.signature(getattr(ref[mod], fn))
            os_ = inspect.signature(getattr(ours[mod], fn))
            rp = [(p.name, p.default) for p in rs.parameters.values()]
            op = [(p.name, p.default) for p in os_.parameters.values()]
            assert [n for n, _ in op[:len(rp)]] == [n for n, _ in rp], (mod, fn, rp, op)
            for (n, d), (_, d2) in zip(rp, op):
                if d is not inspect.Parameter.empty:
                    assert d2 == d or (n == "E" and d2 is None), (mod, fn, n, d, d2)
            for p in list(os_.parameters.values())[len(rp):]:
                assert p.default is not inspect.Parameter.empty, (mod, fn, p.name)
    for meth in ("free_mask_vv", "free_mask_cpl", "local_vv", "apply_S_factorized",
                 "harmonic_extend", "recover_stress", "s_energy", "_local_splits"):
        assert hasattr(condensation.CondensedSystem, meth), meth
    rc = [f.name for f in dataclasses.fields(ref["condensation"].CondensedSystem)]
    for attr in rc:
        assert hasattr(condensation.CondensedSystem, attr) or attr in (
            "fes", "nu", "load", "vv_l2g", "vv_signs", "n_cpl_loc", "nloc_u", "ext_dev",
            "cpl_of_vv", "vv_of_cpl"), attr
    assert dataclasses.asdict(ref["driver"].SolverOptions()) == dataclasses.asdict(D.SolverOptions())
    assert [f.name for f in dataclasses.fields(ref["driver"].SolveResult)] == \
        [f.name for f in dataclasses.fields(D.SolveResult)][:10]


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_apply_S_factorized_matches_reference_S(cuda, name):
    """condensation.py:104-122 vs the reference's assembled S (test_condensation.py:123-143)."""
    g = golden(name)
    prob, fes, sys_ = _system(g)
    S = _csr(g, "S")
    rng = np.random.default_rng(7)
    x = rng.standard_normal(fes.n_vv)
    assert rel(sys_.apply_S_factorized(x), S @ x) <= 1e-12
    xb = np.where(fes.vv_interior, x, 0.0)           # supported on bubbles only
    assert rel(sys_.apply_S_factorized(xb), S @ xb) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_harmonic_extend_matches_reference(cuda, name):
    """condensation.py:93-102 from the reference's own X (ext), and the
    reference's properties: idempotent, energy not above the input's."""
    g = golden(name)
    prob, fes, sys_ = _system(g)
    S = _csr(g, "S")
    x = np.random.default_rng(8).standard_normal(fes.n_vv)
    want = x.copy()
    icpl, iint = sys_._local_splits()
    for t, X in enumerate(g["ext"]):
        loc = x[sys_.vv_l2g[t]] * sys_.vv_signs[t]
        want[sys_.vv_l2g[t][iint]] = -(X @ loc[icpl]) * sys_.vv_signs[t][iint]
    h = sys_.harmonic_extend(x)
    assert rel(h, want) <= 1e-10
    assert np.array_equal(h[~fes.vv_interior], x[~fes.vv_interior])
    assert rel(sys_.harmonic_extend(h), h) <= 1e-12
    assert h @ (S @ h) <= x @ (S @ x) * (1 + 1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_recovery_matrices_match_reference(cuda, name):
    """CondensedSystem.recovery (condensation.py:33,173-177): R_T = M^-1 Bsig^T."""
    g = golden(name)
    prob, fes, sys_ = _system(g)
    R = np.array(sys_.recovery)
    assert R.shape == g["recovery"].shape
    assert rel(R, g["recovery"]) <= 1e-10
    worst = max(rel(a, b) for a, b in zip(R, g["recovery"]))
    assert worst <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_host_attributes_match_reference(cuda, name):
    """Lazy host S / Sd / ext / soo_dense (condensation.py:26-45, 228-238)."""
    g = golden(name)
    prob, fes, sys_ = _system(g)
    assert rel(sys_.S.toarray(), _csr(g, "S").toarray()) <= 1e-12
    assert rel(sys_.Sd.toarray(), _csr(g, "Sd").toarray()) <= 1e-12
    assert rel(np.array(sys_.ext), g["ext"]) <= 1e-10
    assert rel(np.array(sys_.soo_dense), g["soo"]) <= 1e-12
    assert rel(sys_.load, g["load_vv"]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_smoother_from_csr_and_block_list(cuda, name):
    """FacetBlockSmoother(A_csr, blocks, 'jacobi') as the reference builds it
    (driver.py:95-98): the reference's own S_d and block list, against exact
    dense block solves and against the GPU-assembled driver smoother."""
    g = golden(name)
    prob, fes, sys_ = _system(g)
    fc = sys_.free_mask_cpl()
    A = _csr(g, "Sd")[fc][:, fc].tocsr()
    ptr, idx = g["fblk_ptr"], g["fblk_idx"]
    blocks = [idx[ptr[i]:ptr[i + 1]] for i in range(len(ptr) - 1)]
    sm = pc.FacetBlockSmoother(A, blocks, "jacobi")
    r = np.random.default_rng(9).standard_normal(A.shape[0])
    want = np.zeros_like(r)
    for b in blocks:
        want[b] += np.linalg.solve(A[b][:, b].toarray(), r[b])
    assert rel(sm.jacobi_apply(r), want) <= 1e-12
    from paper_2207_08481_b200.operators import SdOperator
    dev = pc.FacetBlockSmoother(SdOperator(sys_), None, "jacobi")
    assert rel(dev.jacobi_apply(r), want) <= 1e-11
    with pytest.raises(NotImplementedError):
        pc.FacetBlockSmoother(A, blocks, "gauss_seidel")
    with pytest.raises(ValueError):
        pc.FacetBlockSmoother(A, blocks, "sor")


@pytest.mark.gpu
@pytest.mark.parametrize("comp", ["additive", "multiplicative"])
def test_asp_from_reference_typed_pieces(cuda, comp):
    """AspPreconditioner(A_csr, smoother, E_c, reference-style CoarseSolver)
    wrapped by ExtendedAsp equals the driver's preconditioner and the
    reference's probe M v (preconditioners.py:286-378)."""
    g = golden("c2_n3")
    prob, fes, sys_ = _system(g)
    fc = sys_.free_mask_cpl()
    A = _csr(g, "Sd")[fc][:, fc].tocsr()
    ptr, idx = g["fblk_ptr"], g["fblk_idx"]
    blocks = [idx[ptr[i]:ptr[i + 1]] for i in range(len(ptr) - 1)]

    class RefCoarse:                      # the reference's CoarseSolver fields
        matrix = _csr(g, "coarse")
        scale = 1.0
        factor = None

    asp = pc.AspPreconditioner(A, pc.FacetBlockSmoother(A, blocks, "jacobi"), _csr(g, "Ec"),
                               RefCoarse(), comp, 1)
    assert asp.jacobi_scale == pytest.approx(float(g[f"jacobi_scale_{comp}"]), rel=1e-10)
    M = pc.ExtendedAsp(sys_, asp)
    assert rel(M(g["probe_v"]), g[f"probe_M_{comp}"]) <= 1e-10


@pytest.mark.gpu
def test_cg_with_reference_style_numpy_callables(cuda):
    """krylov.cg with the reference's operator convention (plain callables on
    NumPy arrays, driver.py:144: `lambda v: S_free @ v`)."""
    from paper_2207_08481_b200.krylov import cg
    g = golden("c2_n3")
    prob, fes, sys_ = _system(g)
    S_free = _csr(g, "S")[fes.vv_free][:, fes.vv_free].tocsr()
    M = D.velocity_preconditioner(fes, sys_, prob.nu,
                                  D.SolverOptions(smoother="jacobi", composition="additive"))
    calls = []

    def apply_A(v):
        calls.append(type(v))
        return S_free @ v

    x, rep = cg(apply_A, g["rhs_u"], lambda v: M(v), rtol=1e-8, maxit=2000)
    assert all(c is np.ndarray for c in calls)
    assert rep.converged and abs(rep.iterations - int(g["cg_additive_iters"])) <= 1
    assert rel(x, g["cg_additive_x"]) <= 1e-7


@pytest.mark.gpu
def test_cg_nan_operator_runs_to_maxit_like_the_reference(cuda):
    """A NaN p'Ap neither raises nor stops (reference krylov.py:121-131):
    the loop runs to maxit and reports not converged, on every launch path."""
    import torch
    from paper_2207_08481_b200 import krylov
    from paper_2207_08481_b200.operators import SOperator
    g = golden("c1_n2")
    prob, fes, sys_ = _system(g)
    M = D.velocity_preconditioner(fes, sys_, prob.nu,
                                  D.SolverOptions(smoother="jacobi", composition="additive"))
    A = SOperator(sys_)
    A.M = torch.full_like(A.M, float("nan"))
    for use_graph in (False, True):
        x, rep = krylov.cg(A, g["rhs_u"], M, rtol=1e-8, maxit=9, use_graph=use_graph)
        assert not rep.converged and rep.iterations == 9
        assert all(np.isnan(r) for r in rep.residuals[1:])
    krylov.release(A)


@pytest.mark.gpu
def test_pcg_state_freed_with_the_operator(cuda):
    """Captured PCG graphs live on the operator: dropping the
    operator frees them; release() frees them at once."""
    import gc
    import weakref
    from paper_2207_08481_b200 import krylov
    from paper_2207_08481_b200.operators import SOperator
    g = golden("c1_n2")
    prob, fes, sys_ = _system(g)
    M = D.velocity_preconditioner(fes, sys_, prob.nu,
                                  D.SolverOptions(smoother="jacobi", composition="additive"))
    A = SOperator(sys_)
    krylov.cg(A, g["rhs_u"], M, rtol=1e-8)
    assert A._pcg_states
    st = weakref.ref(next(iter(A._pcg_states.values())))
    krylov.release(A, M)
    assert not A._pcg_states and st() is None
    krylov.cg(A, g["rhs_u"], M, rtol=1e-8)
    st = weakref.ref(next(iter(A._pcg_states.values())))
    del A
    gc.collect()
    assert st() is None


@pytest.mark.gpu
def test_solve_stokes_elliptic_returns_solve_result(cuda):
    """driver.solve_stokes(mode='elliptic') -> SolveResult with record, p=None,
    sigma, w, checks (driver.py:133-180)."""
    g = golden("c2_n3")
    prob = baseline_config(2, 3)
    opts = D.SolverOptions(mode="elliptic", smoother="jacobi", composition="additive",
                           rtol=1e-8, maxit=2000)
    r = D.solve_stokes(prob, prob.k, prob.nu, opts)
    assert isinstance(r, D.SolveResult) and r.p is None
    assert r.record.iterations == r.report.iterations == int(g["cg_additive_iters"])
    assert r.record.converged and r.record.n_elements == prob.mesh.num_triangles
    assert r.record.max_div == r.checks["max_div_scaled"]
    assert r.sigma is not None and r.w is not None
    assert rel(np.asarray(r.x_free), g["cg_additive_x"]) <= 1e-7
    with pytest.raises(NotImplementedError):            # the reference default smoother
        D.solve_stokes(prob, prob.k, prob.nu, D.SolverOptions(mode="elliptic"))


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present (GPU box)")
def test_integration_install_and_reference_problem_objects():
    """integration.install swaps the reference driver's entry points for the
    GPU ones (and uninstall restores them); the GPU host setup accepts the
    reference's own Problem / Mesh / BoundaryRegions objects and produces the
    same dof maps, geometry and free masks as from this package's mesh."""
    import importlib
    import sys
    sys.path.insert(0, REF_SRC)
    try:
        rdrv = importlib.import_module("mcstokes.driver")
        rmesh = importlib.import_module("mcstokes.mesh")
    finally:
        sys.path.remove(REF_SRC)
    from paper_2207_08481_b200 import integration
    orig = rdrv.solve_stokes
    integration.install(rdrv)
    try:
        assert rdrv.solve_stokes is D.solve_stokes
        assert rdrv.velocity_preconditioner is D.velocity_preconditioner
        assert rdrv.SolverOptions is D.SolverOptions
    finally:
        integration.uninstall(rdrv)
    assert rdrv.solve_stokes is orig
    prob = baseline_config(2, 3)
    m = rmesh.from_arrays(prob.mesh.vertices, prob.mesh.triangles)
    regions = rmesh.classify_boundary(m, dirichlet=lambda x: x[0] < 1 - 1e-12,
                                      neumann=lambda x: x[0] >= 1 - 1e-12)
    ours = FeSystem(prob.mesh, prob.regions, prob.k)
    theirs = FeSystem(m, regions, prob.k)           # the GPU host setup on reference objects
    for a in ("vv_free", "vv_interior", "vv_values", "J", "detJ", "Jinv"):
        assert np.array_equal(getattr(ours, a), getattr(theirs, a)), a
    for a in ("dof_v", "dof_vhat", "dof_vbar", "dof_q"):
        assert np.array_equal(getattr(ours, a).loc2glob, getattr(theirs, a).loc2glob), a
    assert np.array_equal(ours.dof_v.signs, theirs.dof_v.signs)
