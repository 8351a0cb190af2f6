"""Time the k=6 double Schur kernel on the cfg3 condensed S_T (131,072
elements): python tools/ds_bench.py   (MCS_DS6 selects the variant)."""
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
ST, info = engine.condense_gen(k, nt, W, tab)
ext = torch.empty((nt, _abi.call("mcs_ext_stride", k)), dtype=torch.float64, device="cuda")
Sd = torch.empty((nt, _abi.call("mcs_sd_stride", k)), dtype=torch.float64, device="cuda")
def run():
    _abi.call("mcs_double_schur", k, nt, _abi.ptr(ST), _abi.ptr(ext), _abi.ptr(Sd), _abi.ptr(info),
              _abi.stream(None))
for _ in range(3):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ref = Sd[:64].clone()
print(f"MCS_DS6={os.environ.get('MCS_DS6', '0')}: double Schur {np.median(ts):.3f} ms for {nt} "
      f"elements, info {int(info.abs().sum())}, Sd checksum {float(Sd.double().abs().sum()):.12e}")
