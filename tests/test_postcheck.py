"""Post-solve structural checks (reference
driver.py:183-218) against values the reference itself produced on seeded
random velocity / stress vectors (oracle/make_golden.py --postcheck)."""
import numpy as np
import pytest

from conftest import golden
from oracle import mcs_oracle as O
from paper_2207_08481_b200.dofmap import FeSystem
from paper_2207_08481_b200.problems import baseline_config

CASES = [("postcheck_c2_n3", 2, 3), ("postcheck_c3_n2", 3, 2)]


def _fes(cfg, n):
    prob = baseline_config(cfg, n)
    return FeSystem(prob.mesh, prob.regions, prob.k)


@pytest.mark.parametrize("name,cfg,n", CASES)
def test_oracle_post_checks_match_reference(name, cfg, n):
    g = golden(name)
    chk = O.post_checks(_fes(cfg, n), g["u"], g["sigma"], list(g["residuals"]))
    assert abs(chk["max_div_scaled"] - float(g["max_div_scaled"])) <= 1e-12 * float(g["max_div_scaled"])
    assert abs(chk["nt_jump_scaled"] - float(g["nt_jump_scaled"])) <= 1e-12 * float(g["nt_jump_scaled"])
    assert chk["residual_monotone"] == bool(g["residual_monotone"])


@pytest.mark.gpu
@pytest.mark.parametrize("name,cfg,n", CASES)
def test_gpu_post_checks_match_reference(cuda, name, cfg, n):
    from paper_2207_08481_b200.driver import post_checks
    from paper_2207_08481_b200.krylov import KrylovReport
    g = golden(name)
    chk = post_checks(_fes(cfg, n), None, g["u"], g["sigma"],
                      KrylovReport(residuals=list(g["residuals"])))
    np.testing.assert_allclose(chk["max_div_scaled"], float(g["max_div_scaled"]), rtol=1e-12)
    np.testing.assert_allclose(chk["nt_jump_scaled"], float(g["nt_jump_scaled"]), rtol=1e-12)
    assert chk["residual_monotone"] == bool(g["residual_monotone"])
