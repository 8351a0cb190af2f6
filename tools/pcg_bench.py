"""cfg2 PCG solve times (CUDA graphs, median of N solves) for both
compositions: python tools/pcg_bench.py [N]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur  # noqa: E402
from paper_2207_08481_b200.dofmap import FeSystem  # noqa: E402
from paper_2207_08481_b200.driver import SolverOptions, condensed_rhs, velocity_preconditioner  # noqa: E402
from paper_2207_08481_b200.krylov import cg  # noqa: E402
from paper_2207_08481_b200.operators import SOperator  # noqa: E402
from paper_2207_08481_b200.problems import baseline_config  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10
prob = baseline_config(2)
fes = FeSystem(prob.mesh, prob.regions, prob.k)
sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
S = SOperator(sys_)
b = torch.from_numpy(condensed_rhs(fes, sys_)[0]).cuda()
out = {}
for comp in ("additive", "multiplicative"):
    M = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition=comp))
    cg(S, b, M, rtol=1e-8, maxit=2000)
    ts = []
    for _ in range(N):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, rep = cg(S, b, M, rtol=1e-8, maxit=2000)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[comp] = (rep.iterations, float(np.median(ts)), float(np.min(ts)), float(np.max(ts)))
print(os.environ.get("MCS_NO_PDL", "0"), out)
