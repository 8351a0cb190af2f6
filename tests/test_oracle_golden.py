"""The CPU oracle is pinned against golden vectors produced by the reference
itself (oracle/make_golden.py): element blocks, assembled S and S_d, X,
E_c, the coarse matrix, preconditioner applies, jacobi_scale and PCG
iteration counts / solutions."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden, rel
from oracle import mcs_oracle as O
from paper_2207_08481_b200.dofmap import FeSystem
from paper_2207_08481_b200.problems import baseline_config


def csr(g, p):
    return sp.csr_matrix((g[p + "_data"], g[p + "_indices"], g[p + "_indptr"]),
                         shape=tuple(g[p + "_shape"]))


def build(name):
    g = golden(name)
    prob = baseline_config(int(g["cfg"]), int(g["n"]))
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    eb = [O.element_blocks(fes, t, prob.nu, prob.body_force) for t in range(prob.mesh.num_triangles)]
    ST = np.array([O.condense_element(*e[:5])[0] for e in eb])
    return g, prob, fes, eb, O.OracleSystem(fes, prob.nu, ST, np.array([e[5] for e in eb]))


@pytest.mark.parametrize("name", ["c1_n2", "c2_n3", "c3_n2"])
def test_oracle_condensation_matches_reference(name):
    g, prob, fes, eb, s = build(name)
    for i, b in enumerate(("msig", "bws", "bus", "bhs", "adiv")):
        assert rel(np.array([e[i] for e in eb]), g["eb_" + b]) <= 1e-14
    assert rel(s.S.toarray(), csr(g, "S").toarray()) <= 1e-13
    assert rel(s.Sd.toarray(), csr(g, "Sd").toarray()) <= 1e-13
    assert rel(s.X, g["ext"]) <= 1e-13
    assert rel(s.load, g["load_vv"]) <= 1e-14


@pytest.mark.parametrize("name", ["c1_n2", "c2_n3", "c3_n2", "cfg1"])
def test_oracle_pcg_matches_reference(name):
    g, prob, fes, eb, s = build(name)
    assert rel(s.rhs(), g["rhs_u"]) <= 1e-13
    assert rel(s.S_free() @ g["probe_v"], g["probe_Sv"]) <= 1e-13
    assert rel(O.embedding_cpl(fes, s).toarray(), csr(g, "Ec").toarray()) <= 1e-15
    assert rel(O.coarse_matrix(fes, prob.nu).toarray(), csr(g, "coarse").toarray()) <= 1e-15
    for comp in ("additive", "multiplicative"):
        M, asp = O.build_preconditioner(fes, s, prob.nu, comp)
        assert rel(M.apply(g["probe_v"]), g[f"probe_M_{comp}"]) <= 1e-13
        assert asp.scale == pytest.approx(float(g[f"jacobi_scale_{comp}"]), rel=1e-12)
        x, it, res = O.cg(lambda v: s.S_free() @ v, s.rhs(), M.apply, 1e-8, 2000)
        assert it == int(g[f"cg_{comp}_iters"])
        assert rel(x, g[f"cg_{comp}_x"]) <= 1e-10


def test_oracle_microbench_matches_reference():
    g = golden("micro")
    for A, B, S in zip(g["A"], g["B"], g["S"]):
        assert rel(O.spd_schur(A, B), S) <= 1e-14
