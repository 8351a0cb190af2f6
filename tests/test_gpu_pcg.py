"""GPU parity of the PCG hot path (operator apply, ExtendedAsp/ASP
preconditioner, PCG) against the reference's golden outputs and the oracle.
North star: operator applies <= 1e-10 relative l2; PCG iteration count +-1
at rtol 1e-8."""
import numpy as np
import pytest

from conftest import golden, rel
from oracle import mcs_oracle as O
from paper_2207_08481_b200 import preconditioners as pc
from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur
from paper_2207_08481_b200.dofmap import FeSystem
from paper_2207_08481_b200.driver import (SolverOptions, condensed_rhs,
                                           velocity_preconditioner)
from paper_2207_08481_b200.krylov import NegativeCurvatureError, cg
from paper_2207_08481_b200.operators import SdOperator, SOperator
from paper_2207_08481_b200.problems import baseline_config

pytestmark = pytest.mark.gpu
CASES = ["c1_n2", "c2_n3", "c3_n2", "cfg1"]


def _system(g):
    prob = baseline_config(int(g["cfg"]), int(g["n"]))
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
    return prob, fes, sys_


@pytest.mark.parametrize("name", CASES)
def test_operator_apply_matches_reference(cuda, name):
    g = golden(name)
    prob, fes, sys_ = _system(g)
    got = SOperator(sys_)(g["probe_v"])
    assert rel(got, g["probe_Sv"]) <= 1e-10
    assert rel(condensed_rhs(fes, sys_)[0], g["rhs_u"]) <= 1e-12


@pytest.mark.parametrize("name", ["c1_n2", "c2_n3", "c3_n2"])
def test_double_schur_apply_matches_reference(cuda, name):
    import scipy.sparse as sp
    g = golden(name)
    prob, fes, sys_ = _system(g)
    Sd = sp.csr_matrix((g["Sd_data"], g["Sd_indices"], g["Sd_indptr"]),
                       shape=tuple(g["Sd_shape"]))
    fc = sys_.free_mask_cpl()
    Sdf = Sd[fc][:, fc]
    v = np.random.default_rng(3).standard_normal(Sdf.shape[0])
    assert rel(SdOperator(sys_)(v), Sdf @ v) <= 1e-10
    # per-element X against the reference's ext list
    X = np.array(sys_.ext)
    assert rel(X, g["ext"]) <= 1e-12


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("comp", ["additive", "multiplicative"])
def test_preconditioner_apply_matches_reference(cuda, name, comp):
    g = golden(name)
    prob, fes, sys_ = _system(g)
    M = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition=comp))
    assert M.inner.jacobi_scale == pytest.approx(float(g[f"jacobi_scale_{comp}"]), rel=1e-10)
    assert rel(M(g["probe_v"]), g[f"probe_M_{comp}"]) <= 1e-10


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("comp", ["additive", "multiplicative"])
def test_pcg_iterations_match_reference(cuda, name, comp):
    g = golden(name)
    prob, fes, sys_ = _system(g)
    M = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition=comp))
    x, rep = cg(SOperator(sys_), condensed_rhs(fes, sys_)[0], M, rtol=1e-8, maxit=2000)
    ref_it = int(g[f"cg_{comp}_iters"])
    assert rep.converged
    assert abs(rep.iterations - ref_it) <= 1
    assert rel(x, g[f"cg_{comp}_x"]) <= 1e-7
    # residual history tracks the reference's to many digits
    n = min(len(rep.residuals), len(g[f"cg_{comp}_res"]))
    assert np.allclose(rep.residuals[:n], g[f"cg_{comp}_res"][:n], rtol=1e-6, atol=1e-12)


def test_cg_negative_curvature(cuda):
    import torch
    A = np.diag([1.0, -1.0, 2.0])

    def apply_A(v):                # reference convention: NumPy in, NumPy out
        return A @ v

    with pytest.raises(NegativeCurvatureError):
        cg(apply_A, np.array([1.0, 1.0, 1.0]))


def test_cg_zero_rhs(cuda):
    x, rep = cg(lambda v: v, np.zeros(7))
    assert rep.converged and rep.iterations == 0 and not np.any(x)


def test_pcg_bitwise_reproducible(cuda):
    """Run-to-run bitwise identity (the reference's test_cli.py:122-129 idea;
    deterministic scatter + fixed-order reductions)."""
    g = golden("c2_n3")
    prob, fes, sys_ = _system(g)
    M = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition="additive"))
    b = condensed_rhs(fes, sys_)[0]
    x1, r1 = cg(SOperator(sys_), b, M, rtol=1e-8)
    x2, r2 = cg(SOperator(sys_), b, M, rtol=1e-8)
    assert r1.residuals == r2.residuals
    assert np.array_equal(x1, x2)


@pytest.mark.parametrize("comp", ["additive", "multiplicative"])
def test_pcg_two_step_graph_matches_eager(cuda, comp):
    """The two-steps-per-graph loop with its device stop gate against eager
    launches: stopping on the first step of a pair (odd iteration count),
    on the second, and at an odd maxit give the same iterations, residual
    history and x, bit for bit."""
    g = golden("c2_n3")
    prob, fes, sys_ = _system(g)
    M = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition=comp))
    S = SOperator(sys_)
    b = condensed_rhs(fes, sys_)[0]
    _, full = cg(S, b, M, rtol=1e-10, maxit=1000, use_graph=False)
    res = full.residuals
    for parity in (1, 0):     # a new running minimum at an odd / even iteration
        k = next(k for k in range(3, len(res)) if k % 2 == parity and res[k] < min(res[:k]))
        xe, re = cg(S, b, M, rtol=res[k], maxit=1000, use_graph=False)
        xg, rg = cg(S, b, M, rtol=res[k], maxit=1000)
        assert re.iterations == rg.iterations == k and re.converged and rg.converged
        assert re.residuals == rg.residuals and np.array_equal(xe, xg)
    xe, re = cg(S, b, M, rtol=1e-30, maxit=7, use_graph=False)
    xg, rg = cg(S, b, M, rtol=1e-30, maxit=7)
    assert rg.iterations == 7 and not rg.converged
    assert re.residuals == rg.residuals and np.array_equal(xe, xg)


def test_pcg_single_launch_loop_matches_pair_loop(cuda, monkeypatch):
    """The whole PCG loop as one conditional-WHILE graph launch
    (csrc/pcg_loop.cu) against one launch per pair: same iterations,
    residual history and x, bit for bit, including a stop on the first step
    of a pair and a maxit cap below the convergence point."""
    from paper_2207_08481_b200 import krylov
    g = golden("c2_n3")
    prob, fes, sys_ = _system(g)
    M = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition="additive"))
    S = SOperator(sys_)
    b = condensed_rhs(fes, sys_)[0]
    _, full = cg(S, b, M, rtol=1e-10, maxit=1000, use_graph=False)
    res = full.residuals
    k = next(k for k in range(3, len(res)) if k % 2 == 1 and res[k] < min(res[:k]))
    cases = [(1e-8, 1000), (res[k], 1000), (1e-30, 9)]
    out = {}
    for no_loop in (False, True):
        monkeypatch.setattr(krylov, "_NO_LOOP", no_loop)
        krylov.release(S)
        out[no_loop] = [cg(S, b, M, rtol=rt, maxit=mi) for rt, mi in cases]
        st = next(iter(S._pcg_states.values()))
        assert (st.loop is None) == no_loop
        x0, r0 = cg(S, np.zeros_like(b), M)          # b = 0 after the graphs exist
        assert r0.converged and r0.iterations == 0 and not np.any(x0)
        out[no_loop].append(cg(S, b, M, rtol=1e-8, maxit=1000))   # state after b = 0
    krylov.release(S)
    for (xa, ra), (xb, rb) in zip(out[False], out[True]):
        assert ra.iterations == rb.iterations and ra.converged == rb.converged
        assert ra.residuals == rb.residuals and np.array_equal(xa, xb)
    assert out[False][1][1].iterations == k and out[False][2][1].iterations == 9
    assert out[False][3][1].residuals == out[False][0][1].residuals


@pytest.mark.parametrize("cfg,n,leaf", [(1, 16, 48), (2, 40, 128), (3, 24, 96)])
def test_multifrontal_coarse_solve_exact(cuda, cfg, n, leaf):
    """GPU multifrontal triangular solves vs a direct sparse solve."""
    import scipy.sparse.linalg as spla
    from paper_2207_08481_b200 import coarse as co
    prob = baseline_config(cfg, n)
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    A = pc.coarse_matrix(fes, prob.nu)
    xy = fes.mesh.vertices[np.flatnonzero(fes.dof_vbar.is_free) // 2]
    cs = co.factorize_coarse(A, xy, kind="multifrontal", leaf=leaf)
    b = np.random.default_rng(1).standard_normal(A.shape[0])
    ref = spla.spsolve(A.tocsc(), b)
    assert rel(cs.solve(b), ref) <= 1e-12
    # deterministic
    assert np.array_equal(cs.solve(b), cs.solve(b))


@pytest.mark.parametrize("spec", ["1-2", "1-3", "0-1,2-3"])
def test_multifrontal_coarse_solve_exact_with_amalgamated_supernodes(cuda, monkeypatch, spec):
    """Supernode amalgamation of the separator tree (coarse.AMALG): merged
    fronts have more than two children, the level kernels gather one source
    slot per child; the solve stays exact and deterministic."""
    import scipy.sparse.linalg as spla
    from paper_2207_08481_b200 import coarse as co
    prob = baseline_config(2, 40)
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    A = pc.coarse_matrix(fes, prob.nu)
    xy = fes.mesh.vertices[np.flatnonzero(fes.dof_vbar.is_free) // 2]
    monkeypatch.setattr(co, "AMALG", spec)
    monkeypatch.setattr(co, "TOP_MAX", 300)          # keep several levels below the dense top
    cs = co.factorize_coarse(A, xy, kind="multifrontal", leaf=32)
    assert max(len(nd.children) for nd in cs.data.nodes) > 2
    b = np.random.default_rng(2).standard_normal(A.shape[0])
    ref = spla.spsolve(A.tocsc(), b)
    assert rel(cs.solve(b), ref) <= 1e-12
    assert np.array_equal(cs.solve(b), cs.solve(b))
