"""Full GPU pipeline on a BASELINE config: condensation, preconditioner
setup, PCG (both compositions); prints timings and iteration counts."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur  # noqa: E402
from paper_2207_08481_b200.dofmap import FeSystem  # noqa: E402
from paper_2207_08481_b200.driver import SolverOptions, condensed_rhs, velocity_preconditioner  # noqa: E402
from paper_2207_08481_b200.krylov import cg  # noqa: E402
from paper_2207_08481_b200.operators import SOperator  # noqa: E402
from paper_2207_08481_b200.problems import baseline_config  # noqa: E402

cfg = int(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
out = {"cfg": cfg}
t0 = time.perf_counter()
prob = baseline_config(cfg, n)
fes = FeSystem(prob.mesh, prob.regions, prob.k)
out["setup_fes_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
torch.cuda.synchronize()
out["condense_total_s"] = time.perf_counter() - t0
out["elements"] = prob.mesh.num_triangles
out["n_vv_free"] = sys_.maps.n_vv_free
S = SOperator(sys_)
b = torch.from_numpy(condensed_rhs(fes, sys_)[0]).cuda()
for comp in ("additive", "multiplicative"):
    t0 = time.perf_counter()
    M = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition=comp))
    torch.cuda.synchronize()
    t_sup = time.perf_counter() - t0
    t0 = time.perf_counter()
    cg(S, b, M, rtol=1e-8, maxit=3000)
    torch.cuda.synchronize()
    t_first = time.perf_counter() - t0
    times = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, rep = cg(S, b, M, rtol=1e-8, maxit=3000)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    out[comp] = {"iters": rep.iterations, "res": rep.residuals[-1], "solve_ms": float(np.median(times)),
                 "solve_ms_min": min(times),
                 "first_call_incl_capture_s": t_first,
                 "precond_setup_s": t_sup, "jacobi_scale": M.inner.jacobi_scale}
print(json.dumps(out))
