"""Time mcs_condense_gen alone (k = 5, 6; MCS_GEN=1: the CTA-per-element
kernel) and compare S_T with the CTA kernel's.  python tools/gen_bench.py [cfg] [N]"""
import os
import subprocess
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
ST, info = engine.condense_gen(k, nt, W, tab)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); engine.condense_gen(k, nt, W, tab, ST=ST, info=info); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
tag = "cta" if os.environ.get("MCS_GEN") == "1" else "warp-passes"
print(f"k={k} {tag}: condense_gen {np.median(ts):.3f} ms for {nt} elements, info {int(info.abs().sum())}, "
      f"S_T checksum {float(ST.abs().sum()):.13e} first {float(ST[0, 5]):.15e} last {float(ST[-1, -3]):.15e}")
