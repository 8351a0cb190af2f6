"""GPU parity of the batched condensation kernels against the CPU oracle
(north star: relative Frobenius error <= 1e-12 per condensed local matrix)."""
import numpy as np
import pytest

from conftest import golden, rel
from oracle import mcs_oracle as O
from paper_2207_08481_b200 import engine, refblocks
from paper_2207_08481_b200.dofmap import FeSystem
from paper_2207_08481_b200.problems import baseline_config, microbench_host

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _pack_A(A):
    n = A.shape[-1]
    r, c = np.tril_indices(n)
    return np.ascontiguousarray(A[:, r, c])


def test_spd_schur_golden(cuda):
    g = golden("micro")
    A, B, S = g["A"], g["B"], g["S"]
    out, info = engine.spd_schur(60, 36, engine.to_dev(_pack_A(A)), engine.to_dev(B))
    got = engine.unpack_sym(out.cpu().numpy(), 36)
    assert (info.cpu().numpy() == 0).all()
    for i in range(len(A)):
        assert rel(got[i], S[i]) <= TOL


def test_spd_schur_many_elements(cuda):
    A, B = microbench_host(3000, seed=7)
    out, info = engine.spd_schur(60, 36, engine.to_dev(_pack_A(A)), engine.to_dev(B))
    got = engine.unpack_sym(out.cpu().numpy(), 36)
    errs = [rel(got[i], O.spd_schur(A[i], B[i])) for i in range(0, len(A), 7)]
    assert max(errs) <= TOL


def test_spd_schur_not_spd_reports_element(cuda):
    A, B = microbench_host(4, seed=1)
    A[2] = -A[2]
    out, info = engine.spd_schur(60, 36, engine.to_dev(_pack_A(A)), engine.to_dev(B))
    info = info.cpu().numpy()
    assert info[2] == 1 and info[0] == info[1] == info[3] == 0


@pytest.mark.parametrize("cfg,n", [(1, 2), (2, 3), (3, 2), (1, 16)])
def test_condense_matches_oracle(cuda, cfg, n):
    prob = baseline_config(cfg, n)
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    k = prob.k
    refs = refblocks.build_refs(fes)
    W = refblocks.element_weights(fes, prob.nu)
    prog = [engine.to_dev(a) for a in engine.block_program(refs)]
    rec = engine.element_records(len(W), engine.to_dev(W), prog, k)
    blocks = engine.unpack_records(k, rec.cpu().numpy())
    nt = prob.mesh.num_triangles
    sel = range(0, nt, max(1, nt // 40))
    for t in sel:
        ob = O.element_blocks(fes, t, prob.nu)
        for got, ref in zip(blocks, ob[:5]):
            assert rel(got[t], ref) <= 1e-13
    ST, info = engine.condense(k, rec)
    assert (info.cpu().numpy() == 0).all()
    nloc = refblocks.local_sizes(k)["nloc"]
    got = engine.unpack_sym(ST.cpu().numpy(), nloc)
    for t in sel:
        ob = O.element_blocks(fes, t, prob.nu)
        S_ref, _ = O.condense_element(*ob[:5])
        assert rel(got[t], S_ref) <= TOL, (t, rel(got[t], S_ref))


def test_spd_schur_survey_stream_matches_reference(cuda):
    """The first 256 elements of the SURVEY §8d config-5 stream exactly as
    the full-size bench draws it (default_rng(3): G for the whole 65,536
    chunk, then B) against the reference idiom's S (micro_stream.npz)."""
    import torch
    from paper_2207_08481_b200 import engine
    g = golden("micro_stream")
    keep, chunk = int(g["keep"]), int(g["chunk"])
    rng = np.random.default_rng(int(g["seed"]))
    G = rng.standard_normal((chunk, 60, 60))[:keep]
    B = rng.standard_normal((keep, 60, 36))          # = the first keep of the chunk's B
    A = G @ np.swapaxes(G, 1, 2) + 60 * np.eye(60)
    r, c = np.tril_indices(60)
    S = torch.empty((keep, 36 * 37 // 2), dtype=torch.float64, device="cuda")
    info = torch.empty(keep, dtype=torch.int32, device="cuda")
    engine.spd_schur(60, 36, engine.to_dev(np.ascontiguousarray(A[:, r, c])),
                     engine.to_dev(B), out=S, info=info)
    got = engine.unpack_sym(S.cpu().numpy(), 36)
    assert not info.any()
    assert max(rel(got[i], g["S"][i]) for i in range(keep)) <= 1e-12
