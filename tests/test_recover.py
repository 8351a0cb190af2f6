"""Stress recovery: CondensedSystem.recover_stress on the
GPU (csrc/recover.cu) against the reference's -R_T u_T
(condensation.py:64-74, R_T from the LU path of condensation.py:161-177).
The CPU test restates the kernel's structured formula in NumPy."""
import numpy as np
import pytest

from conftest import rel
from oracle import mcs_oracle as O
from paper_2207_08481_b200 import engine, refblocks
from paper_2207_08481_b200.dofmap import FeSystem
from paper_2207_08481_b200.problems import baseline_config

CASES = [(1, 2), (2, 3), (3, 2)]


def _setup(cfg, n):
    prob = baseline_config(cfg, n)
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    return prob, fes


def _oracle(fes, prob, x_full):
    R = []
    for t in range(fes.mesh.num_triangles):
        ob = O.element_blocks(fes, t, prob.nu)
        R.append(O.condense_element(*ob[:5])[1])
    return O.recover_stress(fes, R, x_full)


def structured_recover_np(fes, prob, x_full):
    """NumPy restatement of recover_kernel: sigma_m = Pi_m f_m,
    sigma_b = M_b^-1 f_b, omega = -Phi^-T (d / c), f = Bsig^T u."""
    k = prob.k
    refs = refblocks.build_refs(fes)
    W = refblocks.element_weights(fes, prob.nu)
    ml, nb = k * (k + 1) // 2, 3 * k
    nl = 3 * ml
    Phi = refs.bws[0][:, 0:nl:3]
    l2g, sg = O.vv_maps(fes)
    msig, bws, bus, bhs, _ = refblocks.dense_blocks(refs, W)
    sig, om = [], []
    for t in range(len(W)):
        f = np.vstack([bus[t], bhs[t]]).T @ (x_full[l2g[t]] * sg[t])
        s = W[t, refblocks.W_BWS:refblocks.W_BWS + 3]
        st, r = np.empty(len(f)), np.empty(ml)
        for m in range(ml):
            A = msig[t][3 * m:3 * m + 3, 3 * m:3 * m + 3]
            a, q = np.linalg.solve(A, f[3 * m:3 * m + 3]), np.linalg.solve(A, s)
            r[m] = (s @ a) / (s @ q)
            st[3 * m:3 * m + 3] = a - q * r[m]
        st[nl:] = np.linalg.solve(msig[t][nl:, nl:], f[nl:])
        sig.append(st)
        om.append(-np.linalg.inv(Phi).T @ r)
    return np.concatenate(sig), np.concatenate(om)


@pytest.mark.parametrize("cfg,n", CASES)
def test_structured_recovery_algebra(cfg, n):
    prob, fes = _setup(cfg, n)
    x = np.random.default_rng(11).standard_normal(fes.n_vv)
    s_ref, w_ref = _oracle(fes, prob, x)
    s_np, w_np = structured_recover_np(fes, prob, x)
    assert rel(s_np, s_ref) <= 1e-12
    assert rel(w_np, w_ref) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n", CASES + [(2, 8)])
def test_gpu_recover_stress_matches_oracle(cuda, cfg, n):
    from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur
    prob, fes = _setup(cfg, n)
    sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
    x = np.random.default_rng(12).standard_normal(fes.n_vv)
    sig, om = sys_.recover_stress(x)
    s_ref, w_ref = _oracle(fes, prob, x)
    assert rel(sig, s_ref) <= 1e-10
    assert rel(om, w_ref) <= 1e-10


@pytest.mark.gpu
def test_gpu_recover_stress_device_tensors(cuda):
    import torch
    from paper_2207_08481_b200.condensation import condense_sigma_omega
    prob, fes = _setup(2, 3)
    sys_ = condense_sigma_omega(fes, prob.nu, prob.body_force)
    x = np.random.default_rng(13).standard_normal(fes.n_vv)
    s_h, w_h = sys_.recover_stress(x)
    s_d, w_d = sys_.recover_stress(torch.from_numpy(x).cuda())
    assert np.array_equal(s_d.cpu().numpy(), s_h) and np.array_equal(w_d.cpu().numpy(), w_h)


@pytest.mark.gpu
@pytest.mark.parametrize("name,cfg,n", [("c1_n2", 1, 2), ("c2_n3", 2, 3), ("c3_n2", 3, 2)])
def test_gpu_recover_stress_matches_reference_fixture(cuda, name, cfg, n):
    """Against the recovery matrices R_T the reference itself produced
    (tests/golden, condensation.py:159-177)."""
    from conftest import golden
    from paper_2207_08481_b200.condensation import condense_sigma_omega
    g = golden(name)
    prob, fes = _setup(cfg, n)
    sys_ = condense_sigma_omega(fes, prob.nu, prob.body_force)
    x = np.random.default_rng(14).standard_normal(fes.n_vv)
    sig, om = sys_.recover_stress(x)
    s_ref, w_ref = O.recover_stress(fes, list(g["recovery"]), x)
    assert rel(sig, s_ref) <= 1e-10
    assert rel(om, w_ref) <= 1e-10
