"""cfg2 PCG with a few iterations (for ncu launch lists)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur  # noqa: E402
from paper_2207_08481_b200.dofmap import FeSystem  # noqa: E402
from paper_2207_08481_b200.driver import SolverOptions, condensed_rhs, velocity_preconditioner  # noqa: E402
from paper_2207_08481_b200.krylov import cg  # noqa: E402
from paper_2207_08481_b200.operators import SOperator  # noqa: E402
from paper_2207_08481_b200.problems import baseline_config  # noqa: E402

cfg = int(os.environ.get("PROF_CFG", "2"))
comp = os.environ.get("PROF_COMP", "additive")
prob = baseline_config(cfg)
fes = FeSystem(prob.mesh, prob.regions, prob.k)
sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
M = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition=comp))
S = SOperator(sys_)
b = torch.from_numpy(condensed_rhs(fes, sys_)[0]).cuda()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
x, rep = cg(S, b, M, rtol=1e-8, maxit=int(os.environ.get("PROF_IT", "4")), use_graph=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("iters", rep.iterations)
