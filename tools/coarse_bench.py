"""Time the exact coarse solve alone (CUDA events, warm, graph-free):
python tools/coarse_bench.py [cfg]  (MCS_TOP_MAX overrides the dense-top size)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_08481_b200 import preconditioners as P  # noqa: E402
from paper_2207_08481_b200.dofmap import FeSystem  # noqa: E402
from paper_2207_08481_b200.problems import baseline_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prob = baseline_config(cfg)
fes = FeSystem(prob.mesh, prob.regions, prob.k)
C = P.build_coarse(fes, prob.nu)
n = C.n
b = torch.randn(n, dtype=torch.float64, device="cuda")
x = torch.empty_like(b)
for _ in range(5):
    C.solve_dev(b, x)
torch.cuda.synchronize()
A = C.matrix
res = np.linalg.norm(A @ x.cpu().numpy() - b.cpu().numpy()) / np.linalg.norm(b.cpu().numpy())
ts = []
for _ in range(50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    C.solve_dev(b, x)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    C.solve_dev(b, x)
g.replay()
torch.cuda.synchronize()
tg = []
for _ in range(50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    tg.append(e0.elapsed_time(e1) * 1e3)
print(f"graph replay median {np.median(tg):.1f} us")
d = C.data.dev if C.kind != "dense" else None
print(f"cfg{cfg} n={n} top_t={d['top']['t'] if d else 0} levels={len(d['levels']) if d else 0} "
      f"solve median {np.median(ts):.1f} us min {np.min(ts):.1f} us  rel residual {res:.1e}")
