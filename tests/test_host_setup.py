"""CPU tests: host setup restated from the reference (mesh, bases, dof maps,
reference-matrix element blocks, E_c, coarse matrix, facet blocks,
multifrontal factorisation) pinned against the reference's golden data."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from conftest import golden, rel
from mf_emulate import emulate_hybrid, emulate_solve
from oracle import mcs_oracle as O
from paper_2207_08481_b200 import coarse as co
from paper_2207_08481_b200 import engine, refblocks
from paper_2207_08481_b200 import preconditioners as pc
from paper_2207_08481_b200.dofmap import FeSystem
from paper_2207_08481_b200.maps import element_maps, facet_slots
from paper_2207_08481_b200.problems import baseline_config

CASES = ["c1_n2", "c2_n3", "c3_n2", "cfg1"]


def csr(g, p):
    return sp.csr_matrix((g[p + "_data"], g[p + "_indices"], g[p + "_indptr"]),
                         shape=tuple(g[p + "_shape"]))


def setup(name):
    g = golden(name)
    prob = baseline_config(int(g["cfg"]), int(g["n"]))
    return g, prob, FeSystem(prob.mesh, prob.regions, prob.k)


@pytest.mark.parametrize("name", CASES)
def test_mesh_and_dofs_match_reference(name):
    g, prob, fes = setup(name)
    m = prob.mesh
    assert np.array_equal(m.triangles, g["triangles"])
    for a in ("facets", "facet_tri", "facet_start", "tri_facets"):
        assert np.array_equal(getattr(m, a), g["mesh_" + a]), a
    for a in ("facet_normal", "facet_tangent", "facet_length"):
        assert np.abs(getattr(m, a) - g["mesh_" + a]).max() <= 1e-15
    assert np.array_equal(fes.dof_v.loc2glob, g["v_l2g"])
    assert np.array_equal(fes.dof_v.signs, g["v_signs"])
    assert np.array_equal(fes.dof_vhat.loc2glob, g["h_l2g"])
    assert np.array_equal(fes.dof_vhat.signs, g["h_signs"])
    assert np.array_equal(fes.vv_free, g["vv_free"])
    assert np.array_equal(fes.dof_vbar.is_free, g["vbar_free"])


@pytest.mark.parametrize("name", CASES)
def test_bases_bitwise_equal_reference(name):
    g, prob, fes = setup(name)
    assert np.array_equal(fes.bdm.coef, g["bdm_coef"])
    assert np.array_equal(fes.sigma.coef, g["sigma_coef"])


@pytest.mark.parametrize("name", ["c1_n2", "c2_n3", "c3_n2"])
def test_reference_matrix_blocks_match_quadrature(name):
    g, prob, fes = setup(name)
    refs = refblocks.build_refs(fes)
    W = refblocks.element_weights(fes, prob.nu)
    got = refblocks.dense_blocks(refs, W)
    for blk, key in zip(got, ("msig", "bws", "bus", "bhs", "adiv")):
        for t in range(len(W)):
            assert rel(blk[t], g["eb_" + key][t]) <= 1e-14
    L = refblocks.load_vectors(fes, refs, prob.body_force)
    assert rel(L, g["eb_load"]) <= 1e-14
    assert rel(np.broadcast_to(refs.bpu, g["eb_bpu"].shape), g["eb_bpu"]) <= 1e-14


@pytest.mark.parametrize("name", ["c1_n2", "c2_n3", "c3_n2"])
def test_block_program_reproduces_dense_blocks(name):
    """The sparse (entry -> weight, coef) program walked by the GPU block
    kernel equals the dense weighted sums."""
    g, prob, fes = setup(name)
    refs = refblocks.build_refs(fes)
    W = refblocks.element_weights(fes, prob.nu)
    ptr, widx, coef = engine.block_program(refs)
    rec = np.array([[np.dot(W[t, widx[ptr[q]:ptr[q + 1]]], coef[ptr[q]:ptr[q + 1]])
                     for q in range(len(ptr) - 1)] for t in range(3)])
    want = engine.pack_records(fes.k, *[b[:3] for b in refblocks.dense_blocks(refs, W)])
    assert rel(rec, want) <= 1e-14


@pytest.mark.parametrize("name", CASES)
def test_embedding_cpl_matches_reference(name):
    g, prob, fes = setup(name)

    class S:
        pass
    s = S()
    m = element_maps(fes)
    s.vv_of_cpl, s.cpl_of_vv = m.vv_of_cpl, m.cpl_of_vv
    s.free_mask_cpl = lambda: m.free_cpl
    Ec = pc.embedding_cpl(fes, s)
    assert (abs(Ec - csr(g, "Ec")).max() if Ec.nnz else 0.0) <= 1e-15


@pytest.mark.parametrize("name", ["c1_n2", "c2_n3"])
def test_full_embedding_interior_rows(name):
    """Interior bubble rows of E: the reference's per-element fit, batched."""
    import sys
    g, prob, fes = setup(name)
    E = pc.build_embedding(fes)
    # E reproduces P1 fields exactly (reference test_preconditioners.py:60-74)
    vb = np.zeros(fes.dof_vbar.ndof)
    X = fes.mesh.vertices
    vb[0::2] = 0.3 + X[:, 0] - 2 * X[:, 1]
    vb[1::2] = 1.0 - X[:, 0] + 0.5 * X[:, 1]
    x = E @ vb
    for t in range(fes.mesh.num_triangles):
        uloc = x[:fes.n_v][fes.dof_v.loc2glob[t]] * fes.dof_v.signs[t]
        uv = np.einsum("u,upi->pi", uloc, np.einsum("ij,upj->upi", fes.J[t], fes.tab_u) / fes.detJ[t])
        pts = fes.phys_points(t)
        ue = np.stack([0.3 + pts[:, 0] - 2 * pts[:, 1], 1.0 - pts[:, 0] + 0.5 * pts[:, 1]], 1)
        assert np.abs(uv - ue).max() < 1e-12


@pytest.mark.parametrize("name", CASES)
def test_coarse_matrix_matches_reference(name):
    g, prob, fes = setup(name)
    A = pc.coarse_matrix(fes, prob.nu)
    assert rel(A.toarray(), csr(g, "coarse").toarray()) <= 1e-15


@pytest.mark.parametrize("name", CASES)
def test_facet_blocks_match_reference(name):
    g, prob, fes = setup(name)
    m = element_maps(fes)
    slots, fid = facet_slots(fes, m)
    assert len(fid) == len(g["fblk_ptr"]) - 1


@pytest.mark.parametrize("cfg,n,leaf", [(1, 16, 64), (3, 12, 48), (2, 24, 64)])
def test_multifrontal_factor_exact(cfg, n, leaf):
    """Host emulation of the GPU multifrontal solve schedule equals spsolve."""
    prob = baseline_config(cfg, n)
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    A = pc.coarse_matrix(fes, prob.nu)
    xy = fes.mesh.vertices[np.flatnonzero(fes.dof_vbar.is_free) // 2]
    F = co.multifrontal_factor(A, xy, leaf=leaf)
    b = np.random.default_rng(0).standard_normal(A.shape[0])
    x = emulate_solve(F, b)
    ref = spla.spsolve(A.tocsc(), b)
    assert np.abs(x - ref).max() <= 1e-12 * np.abs(ref).max()
    # with the dense top of the tree (what the GPU runs), small top budget
    co_top = co.TOP_MAX
    try:
        co.TOP_MAX = 200
        xh = emulate_hybrid(F, b)
    finally:
        co.TOP_MAX = co_top
    assert np.abs(xh - ref).max() <= 1e-11 * np.abs(ref).max()


@pytest.mark.parametrize("spec", ["1-2", "1-3", "0-1,2-3"])
def test_multifrontal_factor_exact_with_amalgamated_supernodes(spec):
    """Supernode amalgamation of the separator tree (coarse.AMALG) keeps the
    factorisation exact and removes levels from the schedule."""
    prob = baseline_config(2, 24)
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    A = pc.coarse_matrix(fes, prob.nu)
    xy = fes.mesh.vertices[np.flatnonzero(fes.dof_vbar.is_free) // 2]
    base = co.multifrontal_factor(A, xy, leaf=16)
    keep = co.AMALG
    try:
        co.AMALG = spec
        F = co.multifrontal_factor(A, xy, leaf=16)
    finally:
        co.AMALG = keep
    assert len(F.levels) < len(base.levels)
    assert sorted(F.perm.tolist()) == list(range(A.shape[0]))
    b = np.random.default_rng(1).standard_normal(A.shape[0])
    ref = spla.spsolve(A.tocsc(), b)
    assert np.abs(emulate_solve(F, b) - ref).max() <= 1e-12 * np.abs(ref).max()
    co_top = co.TOP_MAX
    try:
        co.TOP_MAX = 200
        xh = emulate_hybrid(F, b)
    finally:
        co.TOP_MAX = co_top
    assert np.abs(xh - ref).max() <= 1e-11 * np.abs(ref).max()
