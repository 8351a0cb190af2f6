"""Time the facet-block Jacobi apply and the condensed S apply alone at cfg2
(CUDA events, L2 flushed before each call): python tools/smoother_bench.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur  # noqa: E402
from paper_2207_08481_b200.dofmap import FeSystem  # noqa: E402
from paper_2207_08481_b200.driver import SolverOptions, velocity_preconditioner  # noqa: E402
from paper_2207_08481_b200.problems import baseline_config  # noqa: E402

prob = baseline_config(2)
fes = FeSystem(prob.mesh, prob.regions, prob.k)
sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
M = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition="additive"))
sm = M.inner.smoother
nc = sys_.maps.n_cpl_free
r = torch.randn(nc, dtype=torch.float64, device="cuda")
x = torch.empty_like(r)
flush = torch.empty(256 * 2 ** 17, dtype=torch.float64, device="cuda")
flush_rd = torch.ones(256 * 2 ** 17, dtype=torch.float64, device="cuda")   # as bench.py l2_flush
for _ in range(5):
    sm.jacobi_apply(r, out=x)
ts = []
for i in range(50):
    flush.fill_(float(i))
    flush_rd.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sm.jacobi_apply(r, out=x)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
k = prob.k
b = 2 * k + 1
byt = sm.nblk * 8 * b * (b + 1) / 2 + 16 * nc
t = float(np.median(ts))
print(f"variant {os.environ.get('MCS_JAC_VARIANT', '0')}: jacobi {t:.2f} us  "
      f"{byt / t / 1e3:.0f} GB/s  ({byt / t / 1e3 / 6537:.2f} of HBM)")

# condensed S apply (A6) alone, same protocol (bench.py apply_ms)
from paper_2207_08481_b200.operators import SOperator  # noqa: E402
S = SOperator(sys_)
xs = torch.randn(sys_.maps.n_vv_free, dtype=torch.float64, device="cuda")
ys = torch.empty_like(xs)
for _ in range(5):
    S.apply(xs, out=ys)
ta = []
for i in range(50):
    flush.fill_(float(i))
    flush_rd.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    S.apply(xs, out=ys)
    e1.record()
    torch.cuda.synchronize()
    ta.append(e0.elapsed_time(e1) * 1e3)
t = float(np.median(ta))
print(f"S apply {t:.2f} us")
