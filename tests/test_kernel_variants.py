"""The element kernels have A/B variants behind environment switches
 and alternative entry points; all of them must produce the
same matrices.  The switches are read once per process, so each variant runs
in its own interpreter and hands back its outputs as an .npz.

* k = 5, 6: `mcs_condense_fused` (the double Schur as phase D of the passes
  pipeline) against `mcs_condense_gen` + `mcs_double_schur` -- bitwise equal;
* `MCS_GEN=1` (CTA-per-element condensation), `MCS_DS=1` / `MCS_DS=5`
  (shared-memory warp kernel, v5 CTA engine), `MCS_DSR_PAIR=0` against the
  defaults: relative Frobenius <= 1e-12 per array (the north-star tolerance
  for condensed local matrices);
* the config-5 microbench on the one-warp, two-warp and v5 engines against
  the oracle's S = B^T A^-1 B (condensation.py:216-224 idiom): <= 1e-12.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CONDENSE = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2207_08481_b200 import _abi, engine, refblocks
from paper_2207_08481_b200.dofmap import FeSystem
from paper_2207_08481_b200.problems import baseline_config
k, fused, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
prob = baseline_config(3, 5)
fes = FeSystem(prob.mesh, prob.regions, k)
nt = prob.mesh.num_triangles
W = engine.to_dev(refblocks.element_weights(fes, prob.nu))
tab = engine.to_dev(engine.fused_tables(refblocks.build_refs(fes))[0])
mk = lambda n: torch.zeros((nt, n), dtype=torch.float64, device="cuda")
ST, ext, Sd = mk(engine.st_stride(k)), mk(_abi.call("mcs_ext_stride", k)), mk(_abi.call("mcs_sd_stride", k))
info = torch.zeros(nt, dtype=torch.int32, device="cuda")
st = _abi.stream(None)
if fused:
    _abi.call("mcs_condense_fused", k, nt, _abi.ptr(W), W.shape[1], _abi.ptr(tab), _abi.ptr(ST),
              _abi.ptr(ext), _abi.ptr(Sd), _abi.ptr(info), st)
else:
    _abi.call("mcs_condense_gen", k, nt, _abi.ptr(W), W.shape[1], _abi.ptr(tab), _abi.ptr(ST),
              _abi.ptr(info), st)
    _abi.call("mcs_double_schur", k, nt, _abi.ptr(ST), _abi.ptr(ext), _abi.ptr(Sd), _abi.ptr(info), st)
torch.cuda.synchronize()
np.savez(out, ST=ST.cpu().numpy(), ext=ext.cpu().numpy(), Sd=Sd.cpu().numpy(), info=info.cpu().numpy())
"""

_MICRO = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2207_08481_b200 import engine
out = sys.argv[1]
n, m, count = 60, 36, 37        # not a multiple of the CTA width
rng = np.random.default_rng(5)
G = rng.standard_normal((count, n, n))
A = G @ G.transpose(0, 2, 1) + n * np.eye(n)
B = rng.standard_normal((count, n, m))
r, c = np.tril_indices(n)
S = engine.spd_schur(n, m, engine.to_dev(np.ascontiguousarray(A[:, r, c])), engine.to_dev(B))
S = S[0] if isinstance(S, tuple) else S
torch.cuda.synchronize()
np.savez(out, S=S.cpu().numpy(), A=A, B=B)
"""


def _run(script, args, env, tmp_path, name):
    out = str(tmp_path / f"{name}.npz")
    e = dict(os.environ)
    e.update(env)
    p = subprocess.run([sys.executable, "-c", script.format(root=ROOT), *map(str, args), out],
                       env=e, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return np.load(out)


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("k", [5, 6])
def test_phase_d_of_the_passes_pipeline_equals_two_kernels(cuda, tmp_path, k):
    two = _run(_CONDENSE, (k, 0), {}, tmp_path, "two")
    one = _run(_CONDENSE, (k, 1), {}, tmp_path, "one")
    assert not two["info"].any() and not one["info"].any()
    for key in ("ST", "ext", "Sd"):
        assert np.array_equal(two[key], one[key]), key


@pytest.mark.parametrize("k,env", [(6, {"MCS_GEN": "1"}), (5, {"MCS_GEN": "1"}),
                                   (6, {"MCS_DS": "1"}), (6, {"MCS_DS": "5"}),
                                   (5, {"MCS_DS": "1"}), (6, {"MCS_DSR_PAIR": "0"}),
                                   (4, {"MCS_DS": "1"}), (3, {"MCS_DS": "5"})])
def test_condensation_variants_agree(cuda, tmp_path, k, env):
    ref = _run(_CONDENSE, (k, 0), {}, tmp_path, "ref")
    var = _run(_CONDENSE, (k, 0), env, tmp_path, "var")
    assert not ref["info"].any() and not var["info"].any()
    for key in ("ST", "ext", "Sd"):
        assert _rel(var[key], ref[key]) <= 1e-12, (key, env)


@pytest.mark.parametrize("env", [{}, {"MCS_MICRO": "2"}, {"MCS_MICRO": "3"}, {"MCS_MICRO": "5"}])
def test_microbench_engines_match_the_reference_idiom(cuda, tmp_path, env):
    from oracle import mcs_oracle as O
    from paper_2207_08481_b200 import engine
    d = _run(_MICRO, (), env, tmp_path, "micro")
    worst = max(_rel(engine.unpack_sym(d["S"][i], 36), O.spd_schur(d["A"][i], d["B"][i]))
                for i in range(d["A"].shape[0]))
    assert worst <= 1e-12, (env, worst)
