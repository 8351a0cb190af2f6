"""Small driver for ncu captures: one launch of each hot kernel on the
bench workloads (cfg2 condensation pipeline, apply, PCG pieces, microbench)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_08481_b200 import engine, refblocks  # noqa: E402
from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur  # noqa: E402
from paper_2207_08481_b200.dofmap import FeSystem  # noqa: E402
from paper_2207_08481_b200.driver import SolverOptions, condensed_rhs, velocity_preconditioner  # noqa: E402
from paper_2207_08481_b200.krylov import cg  # noqa: E402
from paper_2207_08481_b200.operators import SOperator  # noqa: E402
from paper_2207_08481_b200.problems import baseline_config  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
n = int(os.environ.get("PROF_N", "128"))
if what in ("all", "micro"):
    cnt = int(os.environ.get("PROF_MICRO", str(1 << 16)))
    g = torch.Generator(device="cuda"); g.manual_seed(3)
    G = torch.randn((cnt, 60, 60), dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn((cnt, 60, 36), dtype=torch.float64, device="cuda", generator=g)
    A = torch.bmm(G, G.transpose(1, 2)) + 60 * torch.eye(60, dtype=torch.float64, device="cuda")
    r, c = torch.tril_indices(60, 60, device="cuda")
    Ap = A[:, r, c].contiguous()
    del G, A
    for _ in range(2):
        engine.spd_schur(60, 36, Ap, B)
    torch.cuda.synchronize()
if what in ("all", "cfg"):
    cfg = int(os.environ.get("PROF_CFG", "2"))
    prob = baseline_config(cfg, n if cfg == 2 else None)
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
    M = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition=os.environ.get("PROF_COMP", "multiplicative")))
    x, rep = cg(SOperator(sys_), condensed_rhs(fes, sys_)[0], M, rtol=1e-8, maxit=3)
    torch.cuda.synchronize()
    print("iters", rep.iterations)
if what in ("all", "ds"):
    # cfg3 (k = 6): generation-fused condensation + the warp-per-element double Schur
    prob = baseline_config(3, int(os.environ.get("PROF_N3", "256")))
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
    torch.cuda.synchronize()
    print("cfg3 elements", prob.mesh.num_triangles)
