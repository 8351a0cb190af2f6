"""cfg3 condensation step: condense_gen + mcs_double_schur (two kernels) vs
the fused condense_gen_ds (one kernel); python tools/gen_ds_bench.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_08481_b200 import _abi, engine, refblocks  # noqa: E402
from paper_2207_08481_b200.dofmap import FeSystem  # noqa: E402
from paper_2207_08481_b200.problems import baseline_config  # noqa: E402

prob = baseline_config(3, int(os.environ.get("N", 256)))
fes = FeSystem(prob.mesh, prob.regions, prob.k)
k, nt = prob.k, prob.mesh.num_triangles
refs = refblocks.build_refs(fes)
W = engine.to_dev(refblocks.element_weights(fes, prob.nu))
tab = engine.to_dev(engine.fused_tables(refs)[0])
ST, ext, Sd, info = engine.condense_gen_ds(k, nt, W, tab)
ST2 = torch.empty_like(ST); ext2 = torch.empty_like(ext); Sd2 = torch.empty_like(Sd)
st = _abi.stream(None)


def two():
    _abi.call("mcs_condense_gen", k, nt, _abi.ptr(W), W.shape[1], _abi.ptr(tab), _abi.ptr(ST2),
              _abi.ptr(info), st)
    _abi.call("mcs_double_schur", k, nt, _abi.ptr(ST2), _abi.ptr(ext2), _abi.ptr(Sd2),
              _abi.ptr(info), st)


def one():
    _abi.call("mcs_condense_gen_ds", k, nt, _abi.ptr(W), W.shape[1], _abi.ptr(tab), _abi.ptr(ST),
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


ta, tb = t(two), t(one)
d = [float((a - b).abs().max() / b.abs().max()) for a, b in ((ST2, ST), (ext2, ext), (Sd2, Sd))]
print(f"cfg3 {nt} elements: gen + double_schur {ta:.3f} ms, fused gen_ds {tb:.3f} ms, "
      f"max rel diff S_T/ext/Sd {d}, info {int(info.abs().sum())}")
