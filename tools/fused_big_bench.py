"""cfg3 (k = 6; K=5 via env) condensation: mcs_condense_gen + mcs_double_schur
(two kernels) vs mcs_condense_fused (the passes pipeline with the double Schur
as phase D).  python tools/fused_big_bench.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_08481_b200 import _abi, engine, refblocks  # noqa: E402
from paper_2207_08481_b200.dofmap import FeSystem  # noqa: E402
from paper_2207_08481_b200.problems import baseline_config  # noqa: E402

prob = baseline_config(3, int(os.environ.get("N", 256)))
k = int(os.environ.get("K", prob.k))
fes = FeSystem(prob.mesh, prob.regions, k)
nt = prob.mesh.num_triangles
refs = refblocks.build_refs(fes)
W = engine.to_dev(refblocks.element_weights(fes, prob.nu))
tab = engine.to_dev(engine.fused_tables(refs)[0])
mk = lambda n: torch.empty((nt, n), dtype=torch.float64, device="cuda")
ST, ST2 = mk(engine.st_stride(k)), mk(engine.st_stride(k))
ext, ext2 = mk(_abi.call("mcs_ext_stride", k)), mk(_abi.call("mcs_ext_stride", k))
Sd, Sd2 = mk(_abi.call("mcs_sd_stride", k)), mk(_abi.call("mcs_sd_stride", k))
for a in (ST, ST2, ext, ext2, Sd, Sd2):
    a.zero_()
info = torch.empty(nt, dtype=torch.int32, device="cuda")
st = _abi.stream(None)


def two():
    _abi.call("mcs_condense_gen", k, nt, _abi.ptr(W), W.shape[1], _abi.ptr(tab), _abi.ptr(ST2),
              _abi.ptr(info), st)
    _abi.call("mcs_double_schur", k, nt, _abi.ptr(ST2), _abi.ptr(ext2), _abi.ptr(Sd2),
              _abi.ptr(info), st)


def one():
    _abi.call("mcs_condense_fused", k, nt, _abi.ptr(W), W.shape[1], _abi.ptr(tab), _abi.ptr(ST),
              _abi.ptr(ext), _abi.ptr(Sd), _abi.ptr(info), st)


def t(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


ta = t(two)
i2 = int(info.abs().sum())
tb = t(one)
d = [float((a - b).abs().max() / b.abs().max()) for a, b in ((ST2, ST), (ext2, ext), (Sd2, Sd))]
print(f"k={k} {nt} elements: gen + double_schur {ta:.3f} ms, fused (phase D) {tb:.3f} ms, "
      f"max rel diff S_T/ext/Sd {d}, info {i2} / {int(info.abs().sum())}")
