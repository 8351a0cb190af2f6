"""Drop-in PCG (reference `krylov.py:103-137`) running on the GPU.

Same control flow as the reference: x0 = 0, r = b, z = M r, p = z; per step
Ap, p'Ap (NegativeCurvatureError if <= 0), alpha = rz / p'Ap, x += alpha p,
r -= alpha Ap, recursive residual ||r|| / ||b|| against rtol, z = M r,
beta = rz_new / rz.  `iterations` counts A-applications.

Vectors stay in HBM; the scalars alpha/beta are formed on the device by the
kernels that consume them (blas1.cu) and the host reads back 16 bytes per
iteration (p'Ap and ||r||^2) for the stopping test, exactly the decision
points of the reference loop.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi
from .operators import Workspace, as_device, empty, workspace


class NegativeCurvatureError(Exception):
    """CG met p' A p <= 0: the operator (or preconditioner) is not SPD."""


@dataclass
class KrylovReport:
    iterations: int = 0
    residuals: List[float] = field(default_factory=list)
    converged: bool = False
    lambda_min: Optional[float] = None
    lambda_max: Optional[float] = None
    cond: Optional[float] = None
    lanczos_steps: Optional[int] = None


def _apply(op, v, out):
    if hasattr(op, "apply"):
        return op.apply(v, out=out)
    res = op(v)
    out.copy_(res)
    return out


def cg(apply_A, b, apply_M=None, rtol=1e-8, maxit=1000, stream=None):
    """Preconditioned CG.  `apply_A` / `apply_M` are device operators
    (objects with `.apply(v, out=)`, or callables on CUDA tensors).  `b` may
    be NumPy (returns NumPy) or a CUDA tensor (returns a CUDA tensor)."""
    torch = __import__("torch")
    bd, host = as_device(b)
    n = bd.numel()
    ws: Workspace = workspace()
    sc = ws.sc
    st = _abi.stream(stream)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    r = bd.clone()
    ws.dot(bd, bd, ws.BB)
    bb = float(sc[ws.BB].item())
    report = KrylovReport(residuals=[1.0])
    if bb == 0.0:
        report.converged = True
        return (x.cpu().numpy() if host else x), report
    bnorm = np.sqrt(bb)
    z, Ap = empty(n), empty(n)
    if apply_M is None:
        z.copy_(r)
    else:
        _apply(apply_M, r, z)
    p = z.clone()
    rz, rz_new = ws.RZ0, ws.RZ1
    ws.dot(r, z, rz)
    for it in range(1, maxit + 1):
        _apply(apply_A, p, Ap)
        ws.dot(p, Ap, ws.PAP)
        _abi.call("mcs_cg_update", n, _abi.ptr(x), _abi.ptr(r), _abi.ptr(p), _abi.ptr(Ap),
                  _abi.ptr(sc), rz, ws.PAP, ws.RR, _abi.ptr(ws.partials),
                  _abi.ptr(ws.counter), st)
        pap, rr = sc[ws.PAP:ws.RR + 1].tolist()
        if pap <= 0:
            raise NegativeCurvatureError(f"p'Ap = {pap:.3e} at iteration {it}")
        res = float(np.sqrt(rr) / bnorm)
        report.residuals.append(res)
        report.iterations = it
        if res <= rtol:
            report.converged = True
            break
        if apply_M is None:
            z.copy_(r)
        else:
            _apply(apply_M, r, z)
        ws.dot(r, z, rz_new)
        _abi.call("mcs_xpby", n, _abi.ptr(z), _abi.ptr(p), _abi.ptr(sc), rz_new, rz, st)
        rz, rz_new = rz_new, rz
    return (x.cpu().numpy() if host else x), report
