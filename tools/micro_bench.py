"""Time the config-5 microbench kernel alone (1,048,576 elements, device
inputs from torch's generator) and check a sample against the oracle.
    python tools/micro_bench.py [count]     (MCS_MICRO_V5=1: the v5 engine)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import mcs_oracle as O  # noqa: E402
from paper_2207_08481_b200 import engine  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n, m = 60, 36
g = torch.Generator(device="cuda")
g.manual_seed(3)
Ap = torch.empty((count, n * (n + 1) // 2), dtype=torch.float64, device="cuda")
B = torch.empty((count, n, m), dtype=torch.float64, device="cuda")
r, c = torch.tril_indices(n, n, device="cuda")
eye = n * torch.eye(n, dtype=torch.float64, device="cuda")
for s in range(0, count, 65536):
    e = min(count, s + 65536)
    G = torch.randn((e - s, n, n), dtype=torch.float64, device="cuda", generator=g)
    B[s:e] = torch.randn((e - s, n, m), dtype=torch.float64, device="cuda", generator=g)
    Ap[s:e] = (torch.bmm(G, G.transpose(1, 2)) + eye)[:, r, c]
S = torch.empty((count, m * (m + 1) // 2), dtype=torch.float64, device="cuda")
info = torch.empty(count, dtype=torch.int32, device="cuda")
for _ in range(3):
    engine.spd_schur(n, m, Ap, B, out=S, info=info)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    engine.spd_schur(n, m, Ap, B, out=S, info=info)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = float(np.median(ts))
fl = n ** 3 / 3 + n * n * m + m * m * n
idx = np.random.default_rng(4).choice(count, 32, replace=False)
worst = max(np.linalg.norm(engine.unpack_sym(S[i].cpu().numpy(), m)
                           - O.spd_schur(engine.unpack_sym(Ap[i].cpu().numpy(), n), B[i].cpu().numpy()))
            / np.linalg.norm(O.spd_schur(engine.unpack_sym(Ap[i].cpu().numpy(), n), B[i].cpu().numpy()))
            for i in idx)
print(f"{'v5' if os.environ.get('MCS_MICRO_V5') == '1' else 'w2'}: {t:.3f} ms, "
      f"{count / t / 1e3:.2f} M el/s, {fl * count / t / 1e9:.2f} TF/s "
      f"({fl * count / t / 1e9 / 37.092:.1%} of 37.09), failed {int((info != 0).sum())}, "
      f"max rel err {worst:.1e}")
