"""Stokes (saddle-point) mode: the B / B^T operators, the
block triangular saddle preconditioner and right-preconditioned GMRES
(reference driver.py:148-160, preconditioners.py:384-420, krylov.py:25-100)
against fixtures produced by the reference itself (oracle/make_golden.py
--stokes).  CPU tests pin the oracle restatement; GPU tests run the device
path through the C ABI."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden, rel
from oracle import mcs_oracle as O
from paper_2207_08481_b200 import refblocks
from paper_2207_08481_b200.dofmap import FeSystem
from paper_2207_08481_b200.problems import baseline_config

CASES = [("stokes_c1_n2", 1, 2), ("stokes_c2_n3", 2, 3), ("stokes_c3_n2", 3, 2)]


def _csr(g, prefix):
    return sp.csr_matrix((g[prefix + "_data"], g[prefix + "_indices"], g[prefix + "_indptr"]),
                         shape=tuple(g[prefix + "_shape"]))


def _setup(cfg, n):
    prob = baseline_config(cfg, n)
    return prob, FeSystem(prob.mesh, prob.regions, prob.k)


@pytest.mark.parametrize("name,cfg,n", CASES)
def test_oracle_B_matches_reference(name, cfg, n):
    g = golden(name)
    prob, fes = _setup(cfg, n)
    B = O.assemble_B(fes, refblocks.build_refs(fes).bpu)
    assert rel(B.toarray(), _csr(g, "B").toarray()) <= 1e-13


@pytest.mark.parametrize("name,cfg,n", CASES[:2])
def test_oracle_gmres_reproduces_reference(name, cfg, n):
    g = golden(name)
    prob, fes = _setup(cfg, n)
    eb = [O.element_blocks(fes, t, prob.nu, prob.body_force) for t in range(fes.mesh.num_triangles)]
    osys = O.OracleSystem(fes, prob.nu, np.array([O.condense_element(*b[:5])[0] for b in eb]),
                          np.array([b[5] for b in eb]))
    free = fes.vv_free
    B_free = O.assemble_B(fes, refblocks.build_refs(fes).bpu)[:, free].tocsr()
    K = sp.bmat([[osys.S_free(), B_free.T], [B_free, None]], format="csr")
    assert rel(K @ g["probe_v"], g["probe_Kv"]) <= 1e-13
    diag = O.pressure_mass_diag(fes, prob.nu)
    for comp in ("additive", "multiplicative"):
        M, _ = O.build_preconditioner(fes, osys, prob.nu, comp)
        P = O.saddle_apply(M.apply, diag, B_free)
        assert rel(P(g["probe_v"]), g[f"probe_P_{comp}"]) <= 1e-12
        x, it, res = O.gmres(lambda u: K @ u, g["rhs"], P, rtol=1e-8, maxit=500)
        assert it == int(g[f"gmres_{comp}_iters"])
        assert rel(x, g[f"gmres_{comp}_x"]) <= 1e-9


# ----------------------------------------------------------------- GPU


def _gpu_system(cfg, n):
    from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur
    prob, fes = _setup(cfg, n)
    sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
    return prob, fes, sys_


@pytest.mark.gpu
@pytest.mark.parametrize("name,cfg,n", CASES)
def test_gpu_saddle_operator_and_preconditioner(cuda, name, cfg, n):
    from paper_2207_08481_b200 import preconditioners as pc
    from paper_2207_08481_b200.driver import SolverOptions, velocity_preconditioner
    from paper_2207_08481_b200.operators import SaddleOperator
    g = golden(name)
    prob, fes, sys_ = _gpu_system(cfg, n)
    K = SaddleOperator(sys_)
    assert rel(K(g["probe_v"]), g["probe_Kv"]) <= 1e-10
    nv = K.n_v
    Bt = K.B.apply_T(g["probe_v"][nv:])
    assert rel(Bt, _csr(g, "B")[:, fes.vv_free].T @ g["probe_v"][nv:]) <= 1e-12
    mp = pc.PressureMassPrecond.build(fes, prob.nu)
    for comp in ("additive", "multiplicative"):
        vel = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition=comp))
        P = pc.SaddlePreconditioner(vel, mp, K.B)
        assert rel(P(g["probe_v"]), g[f"probe_P_{comp}"]) <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("name,cfg,n", CASES)
def test_gpu_gmres_matches_reference(cuda, name, cfg, n):
    from paper_2207_08481_b200 import preconditioners as pc
    from paper_2207_08481_b200.driver import SolverOptions, condensed_rhs, velocity_preconditioner
    from paper_2207_08481_b200.krylov import gmres
    from paper_2207_08481_b200.operators import SaddleOperator
    g = golden(name)
    prob, fes, sys_ = _gpu_system(cfg, n)
    K = SaddleOperator(sys_)
    rhs = np.concatenate(condensed_rhs(fes, sys_))
    assert rel(rhs, g["rhs"]) <= 1e-12
    mp = pc.PressureMassPrecond.build(fes, prob.nu)
    for comp in ("additive", "multiplicative"):
        vel = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition=comp))
        P = pc.SaddlePreconditioner(vel, mp, K.B)
        x, rep = gmres(K, rhs, P, rtol=1e-8, maxit=500)
        ref_it = int(g[f"gmres_{comp}_iters"])
        assert rep.converged and abs(rep.iterations - ref_it) <= 1, (comp, rep.iterations, ref_it)
        assert rel(x, g[f"gmres_{comp}_x"]) <= 1e-6
        m = min(len(rep.residuals), len(g[f"gmres_{comp}_res"]))
        np.testing.assert_allclose(rep.residuals[:m], g[f"gmres_{comp}_res"][:m], rtol=1e-4,
                                   atol=1e-12)


@pytest.mark.gpu
def test_gpu_solve_stokes_end_to_end(cuda):
    """driver.solve_stokes in Stokes mode: GMRES solution against a direct
    solve of the reference's K, pressure sign convention, stress recovery."""
    import scipy.sparse.linalg as spla
    from paper_2207_08481_b200.driver import SolverOptions, solve_stokes
    g = golden("stokes_c2_n3")
    prob, fes = _setup(2, 3)
    r = solve_stokes(prob, prob.k, prob.nu,
                     SolverOptions(mode="stokes", smoother="jacobi", composition="additive", rtol=1e-10,
                                   maxit=500))
    assert r.report.converged
    free = fes.vv_free
    B_free = _csr(g, "B")[:, free]
    K = sp.bmat([[r.system.S[free][:, free], B_free.T], [B_free, None]], format="csc")
    x = spla.spsolve(K, g["rhs"])
    nv = int(free.sum())
    assert rel(np.asarray(r.x_free), x[:nv]) <= 1e-7
    assert rel(r.p, -x[nv:]) <= 1e-7
    assert r.sigma.shape == (fes.mesh.num_triangles * refblocks.local_sizes(prob.k)["ns"],)
    # reference post_checks on the same (u, sigma, history), restated
    ref = O.post_checks(fes, r.u, r.sigma, r.report.residuals)
    np.testing.assert_allclose(r.checks["max_div_scaled"], ref["max_div_scaled"], rtol=1e-9,
                               atol=1e-14)
    np.testing.assert_allclose(r.checks["nt_jump_scaled"], ref["nt_jump_scaled"], rtol=1e-9,
                               atol=1e-14)
    assert r.checks["max_div_scaled"] < 1e-8          # MCS velocities are divergence-free
