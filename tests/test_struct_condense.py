"""Structured sigma/omega condensation (csrc/condense_struct.cu, DESIGN.md
§3.2): the block structure it relies on holds for the reference's own
element blocks, the compact-record program reproduces the reference blocks,
and S_T = adiv + Y Y^T equals the reference's LU condensation
(condensation.py:161-176) to round-off.  CPU tests restate the kernel's
algebra in NumPy; GPU tests run the kernel through the C ABI."""
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


def _oracle_blocks(fes, prob, elems):
    return [O.element_blocks(fes, t, prob.nu) for t in elems]


def _host_program_eval(prog, W, length):
    ptr, widx, coef = prog
    out = np.zeros((len(W), length))
    for q in range(length):
        for p in range(ptr[q], ptr[q + 1]):
            out[:, q] += W[:, widx[p]] * coef[p]
    return out


def structured_condense_np(rec, k):
    """NumPy restatement of condense_struct_kernel on one compact record."""
    L = engine.srecord_layout(k)
    z = refblocks.local_sizes(k)
    ml, nb, ns, nloc, nu = L["ml"], L["nb"], z["ns"], z["nloc"], z["nu"]
    s = rec[0:3]
    B = rec[L["B"]:L["B"] + nloc * ns].reshape(nloc, ns)
    cols = []
    for m in range(ml):
        A = rec[L["A"] + 9 * m:L["A"] + 9 * m + 9].reshape(3, 3)
        Lm = np.linalg.cholesky(A)
        v = np.linalg.solve(Lm, s)
        u = v / np.linalg.norm(v)
        ax = int(np.argmin(np.abs(u)))
        q1 = -u[ax] * u
        q1[ax] += 1.0
        q1 /= np.linalg.norm(q1)
        Q = np.stack([q1, np.cross(u, q1)], 1)
        cols.append(B[:, 3 * m:3 * m + 3] @ np.linalg.solve(Lm.T, Q))
    Mb = rec[L["Mb"]:L["Mb"] + nb * nb].reshape(nb, nb)
    Lb = np.linalg.cholesky(Mb)
    cols.append(np.linalg.solve(Lb, B[:, 3 * ml:].T).T)
    Y = np.hstack(cols)
    S = Y @ Y.T
    S[:nu, :nu] += rec[L["adiv"]:L["adiv"] + nu * nu].reshape(nu, nu)
    return S


@pytest.mark.parametrize("cfg,n", CASES)
def test_reference_blocks_have_the_structure(cfg, n):
    prob, fes = _setup(cfg, n)
    ob = _oracle_blocks(fes, prob, range(min(8, fes.mesh.num_triangles)))
    msig = np.array([b[0] for b in ob])
    bws = np.array([b[1] for b in ob])
    assert engine.structure_error(msig, bws, prob.k) <= 1e-13


def test_structure_check_rejects_dense_blocks():
    k = 2
    rng = np.random.default_rng(0)
    z = refblocks.local_sizes(k)
    G = rng.standard_normal((1, z["ns"], z["ns"]))
    msig = G @ G.transpose(0, 2, 1) + z["ns"] * np.eye(z["ns"])
    bws = rng.standard_normal((1, z["nw"], z["ns"]))
    assert engine.structure_error(msig, bws, k) > 1e-3


@pytest.mark.parametrize("cfg,n", CASES)
def test_compact_program_matches_reference_blocks(cfg, n):
    prob, fes = _setup(cfg, n)
    k = prob.k
    refs = refblocks.build_refs(fes)
    W = refblocks.element_weights(fes, prob.nu)
    L = engine.srecord_layout(k)
    elems = list(range(0, fes.mesh.num_triangles, max(1, fes.mesh.num_triangles // 6)))
    got = _host_program_eval(engine.sblock_program(refs), W[elems], L["len"])
    ob = _oracle_blocks(fes, prob, elems)
    want = engine.pack_srecords(k, *[np.array([b[i] for b in ob]) for i in range(5)])
    s_got = got[:, 0:3] / np.linalg.norm(got[:, 0:3], axis=1, keepdims=True)
    assert np.allclose(np.abs(np.sum(s_got * want[:, 0:3], 1)), 1.0, atol=1e-14)
    for a, b in zip(got, want):
        assert rel(a[4:], b[4:]) <= 1e-13


@pytest.mark.parametrize("cfg,n", CASES)
def test_structured_algebra_matches_reference_lu(cfg, n):
    prob, fes = _setup(cfg, n)
    nt = fes.mesh.num_triangles
    elems = list(range(0, nt, max(1, nt // 10)))
    ob = _oracle_blocks(fes, prob, elems)
    recs = engine.pack_srecords(prob.k, *[np.array([b[i] for b in ob]) for i in range(5)])
    for rec, b in zip(recs, ob):
        S_ref, _ = O.condense_element(*b[:5])
        assert rel(structured_condense_np(rec, prob.k), S_ref) <= 1e-13


# ----------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n", [(1, 2), (2, 3), (3, 2), (1, 16), (2, 8)])
def test_gpu_structured_condense_matches_oracle(cuda, cfg, n):
    prob, fes = _setup(cfg, n)
    k = prob.k
    refs = refblocks.build_refs(fes)
    W = refblocks.element_weights(fes, prob.nu)
    prog = [engine.to_dev(a) for a in engine.sblock_program(refs)]
    rec = engine.element_srecords(len(W), engine.to_dev(W), prog, k)
    ST, info = engine.condense_struct(k, rec)
    assert (info.cpu().numpy() == 0).all()
    nloc = refblocks.local_sizes(k)["nloc"]
    got = engine.unpack_sym(ST.cpu().numpy(), nloc)
    nt = fes.mesh.num_triangles
    for t in range(0, nt, max(1, nt // 40)):
        ob = O.element_blocks(fes, t, prob.nu)
        S_ref, _ = O.condense_element(*ob[:5])
        assert rel(got[t], S_ref) <= 1e-12, (t, rel(got[t], S_ref))


@pytest.mark.gpu
@pytest.mark.parametrize("k", [2, 3, 4, 5, 6])
def test_gpu_structured_condense_all_degrees(cuda, k):
    """Every compiled degree against the NumPy restatement (random affine
    elements through the host-packed path)."""
    prob = baseline_config(2, 2)
    fes = FeSystem(prob.mesh, prob.regions, k)
    refs = refblocks.build_refs(fes)
    W = refblocks.element_weights(fes, prob.nu)
    L = engine.srecord_layout(k)
    recs = _host_program_eval(engine.sblock_program(refs), W, L["len"])
    ST, info = engine.condense_struct(k, engine.to_dev(recs))
    assert (info.cpu().numpy() == 0).all()
    nloc = refblocks.local_sizes(k)["nloc"]
    got = engine.unpack_sym(ST.cpu().numpy(), nloc)
    for t in range(len(W)):
        assert rel(got[t], structured_condense_np(recs[t], k)) <= 1e-12


@pytest.mark.gpu
def test_gpu_structured_condense_reports_singular_element(cuda):
    prob, fes = _setup(2, 2)
    k = prob.k
    refs = refblocks.build_refs(fes)
    W = refblocks.element_weights(fes, prob.nu)
    L = engine.srecord_layout(k)
    recs = _host_program_eval(engine.sblock_program(refs), W, L["len"])
    recs[3, L["A"] + 9:L["A"] + 18] *= -1.0          # block m=1 of element 3 not SPD
    recs[5, L["Mb"]] = -1.0                           # bubble block of element 5
    _, info = engine.condense_struct(k, engine.to_dev(recs))
    info = info.cpu().numpy()
    assert info[3] != 0 and info[5] != 0
    assert (np.delete(info, [3, 5]) == 0).all()


# ------------------------------------------------------- fused kernel (k <= 4)

def test_fused_tables_reproduce_reference_bsig():
    """Host evaluation of the fused kernel's row formula
    B[i] = base[i] + sum_a W[woff[i] + a] T_a[i] equals the reference's
    [bus; bhs] (assembly.py:66-83)."""
    prob, fes = _setup(2, 3)
    refs = refblocks.build_refs(fes)
    W = refblocks.element_weights(fes, prob.nu)
    tab, woff = engine.fused_tables(refs)
    L = engine.fused_table_layout(prob.k)
    z = refblocks.local_sizes(prob.k)
    NR, ns, nloc = L["NR"], z["ns"], z["nloc"]
    G4 = tab[L["G4"]:L["G4"] + 4 * NR * ns].reshape(NR, ns, 4)
    base, T = G4[..., 0], np.moveaxis(G4[..., 1:], -1, 0)
    Wz = np.concatenate([W, np.zeros((len(W), 6))], 1)
    for t in range(0, fes.mesh.num_triangles, 5):
        B = base + sum(Wz[t, woff + a][:, None] * T[a] for a in range(3))
        ob = O.element_blocks(fes, t, prob.nu)
        assert rel(B[:nloc], np.vstack([ob[2], ob[3]])) <= 1e-13
        assert np.abs(B[nloc:]).max() == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n,k", [(1, 2, 2), (1, 16, 2), (2, 3, 4), (2, 8, 4), (2, 3, 3)])
def test_gpu_fused_matches_oracle(cuda, cfg, n, k):
    prob, _ = _setup(cfg, n)
    fes = FeSystem(prob.mesh, prob.regions, k)
    refs = refblocks.build_refs(fes)
    W = engine.to_dev(refblocks.element_weights(fes, prob.nu))
    tab, _ = engine.fused_tables(refs)
    nt = fes.mesh.num_triangles
    ST, ext, Sd, info = engine.condense_fused(k, nt, W, engine.to_dev(tab))
    assert (info.cpu().numpy() == 0).all()
    z = refblocks.local_sizes(k)
    ni, nc = z["n_int"], z["ncpl"]
    S_got = engine.unpack_sym(ST.cpu().numpy(), z["nloc"])
    E = ext.cpu().numpy()
    Sd_got = engine.unpack_sym(Sd.cpu().numpy(), nc)
    for t in range(0, nt, max(1, nt // 30)):
        ob = O.element_blocks(fes, t, prob.nu)
        S_ref, _ = O.condense_element(*ob[:5])
        assert rel(S_got[t], S_ref) <= 1e-12, ("S_T", t)
        Soo, X, Sd_ref = O.double_schur_element(S_ref, k)
        assert rel(E[t, :ni * nc].reshape(ni, nc), X) <= 1e-12, ("X", t)
        Sinv = engine.unpack_sym(E[t, ni * nc:ni * nc + ni * (ni + 1) // 2], ni)
        assert rel(Sinv, np.linalg.inv(Soo)) <= 1e-12, ("Soo^-1", t)
        assert rel(Sd_got[t], Sd_ref) <= 1e-12, ("Sd", t)


@pytest.mark.gpu
def test_gpu_fused_reports_failures(cuda):
    """A negative-definite geometry weight set makes the stress blocks
    indefinite: bit 0 of info (the reference's 'singular local stress block');
    other elements stay clean."""
    prob, fes = _setup(2, 2)
    refs = refblocks.build_refs(fes)
    W = refblocks.element_weights(fes, prob.nu)
    W[1, refblocks.W_MSIG:refblocks.W_MSIG + 6] *= -1.0
    tab, _ = engine.fused_tables(refs)
    nt = fes.mesh.num_triangles
    _, _, _, info = engine.condense_fused(prob.k, nt, engine.to_dev(W), engine.to_dev(tab))
    info = info.cpu().numpy()
    assert info[1] & 1
    assert (np.delete(info, [1]) == 0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("k", [2, 3, 4, 5, 6])
def test_gpu_double_schur_kernel_matches_oracle(cuda, k):
    """mcs_double_schur (the k = 5, 6 path; v5 engine) on GPU-condensed S_T:
    X, S_oo^-1 and Sd_T against condensation.py:207-226."""
    import torch
    from paper_2207_08481_b200 import _abi
    prob = baseline_config(2, 2)
    fes = FeSystem(prob.mesh, prob.regions, k)
    refs = refblocks.build_refs(fes)
    W = refblocks.element_weights(fes, prob.nu)
    L = engine.srecord_layout(k)
    recs = _host_program_eval(engine.sblock_program(refs), W, L["len"])
    ST, info = engine.condense_struct(k, engine.to_dev(recs))
    nt = len(W)
    ext = torch.empty((nt, _abi.call("mcs_ext_stride", k)), dtype=torch.float64, device="cuda")
    Sd = torch.empty((nt, _abi.call("mcs_sd_stride", k)), dtype=torch.float64, device="cuda")
    _abi.call("mcs_double_schur", k, nt, _abi.ptr(ST), _abi.ptr(ext), _abi.ptr(Sd),
              _abi.ptr(info), _abi.stream(None))
    assert (info.cpu().numpy() == 0).all()
    z = refblocks.local_sizes(k)
    ni, nc = z["n_int"], z["ncpl"]
    S_all = engine.unpack_sym(ST.cpu().numpy(), z["nloc"])
    E = ext.cpu().numpy()
    Sd_got = engine.unpack_sym(Sd.cpu().numpy(), nc)
    for t in range(nt):
        Soo, X, Sd_ref = O.double_schur_element(S_all[t], k)
        assert rel(E[t, :ni * nc].reshape(ni, nc), X) <= 1e-12
        Sinv = engine.unpack_sym(E[t, ni * nc:ni * nc + ni * (ni + 1) // 2], ni)
        assert rel(Sinv, np.linalg.inv(Soo)) <= 1e-12
        assert rel(Sd_got[t], Sd_ref) <= 1e-12


@pytest.mark.gpu
def test_gpu_condensation_edge_cases(cuda):
    """Empty batches are no-ops (return 0, touch nothing); a single element
    and a batch that is not a multiple of the warps per CTA condense like
    the full mesh; the fused kernel is bitwise deterministic run to run."""
    import torch
    prob, fes = _setup(2, 3)
    k = prob.k
    refs = refblocks.build_refs(fes)
    W = refblocks.element_weights(fes, prob.nu)
    tab = engine.to_dev(engine.fused_tables(refs)[0])
    Wd = engine.to_dev(W)
    # empty batch
    ST, ext, Sd, info = engine.condense_fused(k, 0, Wd, tab)
    assert ST.shape[0] == 0 and info.shape[0] == 0
    # full mesh reference
    ST_all, ext_all, Sd_all, _ = engine.condense_fused(k, len(W), Wd, tab)
    z = refblocks.local_sizes(k)
    ne = z["n_int"] * z["ncpl"] + z["n_int"] * (z["n_int"] + 1) // 2   # ext payload (stride is even)
    ext_all = ext_all[:, :ne]
    torch.cuda.synchronize()
    for sub in ([7], list(range(13))):            # single element, ragged batch
        ST_s, ext_s, Sd_s, info_s = engine.condense_fused(k, len(sub), engine.to_dev(W[sub]), tab)
        assert (info_s.cpu().numpy() == 0).all()
        assert torch.equal(ST_s, ST_all[sub]) and torch.equal(ext_s[:, :ne], ext_all[sub])
        assert torch.equal(Sd_s, Sd_all[sub])
    ST2, ext2, Sd2, _ = engine.condense_fused(k, len(W), Wd, tab)
    assert torch.equal(ST2, ST_all) and torch.equal(ext2[:, :ne], ext_all)
    assert torch.equal(Sd2, Sd_all)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n,k", [(2, 3, 4), (2, 3, 5), (3, 2, 6), (3, 4, 6)])
def test_gpu_condense_gen_matches_oracle(cuda, cfg, n, k):
    """Generation-fused structured condensation (the k = 5, 6 path) against
    the reference's LU condensation (condensation.py:161-176)."""
    prob, _ = _setup(cfg, n)
    fes = FeSystem(prob.mesh, prob.regions, k)
    refs = refblocks.build_refs(fes)
    W = engine.to_dev(refblocks.element_weights(fes, prob.nu))
    tab, _ = engine.fused_tables(refs)
    nt = fes.mesh.num_triangles
    ST, info = engine.condense_gen(k, nt, W, engine.to_dev(tab))
    assert (info.cpu().numpy() == 0).all()
    got = engine.unpack_sym(ST.cpu().numpy(), refblocks.local_sizes(k)["nloc"])
    for t in range(0, nt, max(1, nt // 20)):
        ob = O.element_blocks(fes, t, prob.nu)
        S_ref, _ = O.condense_element(*ob[:5])
        assert rel(got[t], S_ref) <= 1e-12, (t, rel(got[t], S_ref))
