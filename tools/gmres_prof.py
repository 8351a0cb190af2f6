"""Stokes GMRES at cfg2: solve time, and with GMRES_IT set a fixed number of
iterations (ncu launch lists: GMRES_IT=40 ncu --metrics gpu__time_duration.sum
... python tools/gmres_prof.py)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_08481_b200 import preconditioners as pc  # noqa: E402
from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur  # noqa: E402
from paper_2207_08481_b200.dofmap import FeSystem  # noqa: E402
from paper_2207_08481_b200.driver import SolverOptions, condensed_rhs, velocity_preconditioner  # noqa: E402
from paper_2207_08481_b200.krylov import _GS_STATS, gmres  # noqa: E402
from paper_2207_08481_b200.operators import SaddleOperator  # noqa: E402
from paper_2207_08481_b200.problems import baseline_config  # noqa: E402

prob = baseline_config(2)
fes = FeSystem(prob.mesh, prob.regions, prob.k)
sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
K = SaddleOperator(sys_)
vel = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition="additive"))
P = pc.SaddlePreconditioner(vel, pc.PressureMassPrecond.build(fes, prob.nu), K.B)
rhs = torch.from_numpy(np.concatenate(condensed_rhs(fes, sys_))).cuda()
it = int(os.environ.get("GMRES_IT", "1000"))
rtol = 1e-8 if it == 1000 else 1e-30
gmres(K, rhs, P, rtol=rtol, maxit=min(it, 20))
torch.cuda.synchronize()
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    x, rep = gmres(K, rhs, P, rtol=rtol, maxit=it)
    e1.record()
    torch.cuda.synchronize()
    print(f"iterations {rep.iterations} device {e0.elapsed_time(e1):.1f} ms wall "
          f"{1e3 * (time.perf_counter() - t0):.1f} ms  per it {e0.elapsed_time(e1) / rep.iterations:.3f} ms")
print("Gram-Schmidt:", _GS_STATS)
