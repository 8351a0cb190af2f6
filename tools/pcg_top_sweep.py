"""cfg2 PCG solve time vs the size of the dense top block of the coarse solve."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_08481_b200 import coarse  # noqa: E402
from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur  # noqa: E402
from paper_2207_08481_b200.dofmap import FeSystem  # noqa: E402
from paper_2207_08481_b200.driver import SolverOptions, condensed_rhs, velocity_preconditioner  # noqa: E402
from paper_2207_08481_b200.krylov import cg  # noqa: E402
from paper_2207_08481_b200.operators import SOperator  # noqa: E402
from paper_2207_08481_b200.problems import baseline_config  # noqa: E402

cfg = int(os.environ.get("PROF_CFG", "2"))
prob = baseline_config(cfg)
fes = FeSystem(prob.mesh, prob.regions, prob.k)
sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
S = SOperator(sys_)
b = torch.from_numpy(condensed_rhs(fes, sys_)[0]).cuda()
for top in [int(v) for v in sys.argv[1:]] or [4096]:
    coarse.TOP_MAX = top
    t0 = time.perf_counter()
    M = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition="additive"))
    setup = time.perf_counter() - t0
    cg(S, b, M, rtol=1e-8, maxit=400)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, rep = cg(S, b, M, rtol=1e-8, maxit=400)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"TOP_MAX={top} iters={rep.iterations} solve_ms={ts[2]:.2f} per_it={ts[2] / rep.iterations:.3f} setup_s={setup:.2f}", flush=True)
