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


def _apply(op, v, out, host_callables=False):
    """out = op(v).  This package's device operators (`.apply(v, out=)`)
    run on the CUDA tensors directly.  Any other callable follows the
    reference convention (krylov.py:25,103: a plain callable v -> A v on 1-D
    float64 arrays): with a NumPy right-hand side it receives and may return
    NumPy arrays, with a CUDA right-hand side it receives the CUDA tensor;
    NumPy or torch results are both accepted."""
    if hasattr(op, "apply"):
        return op.apply(v, out=out)
    res = op(v.cpu().numpy() if host_callables else v)
    if isinstance(res, np.ndarray):
        res = __import__("torch").from_numpy(np.ascontiguousarray(res, dtype=np.float64))
    out.copy_(res)
    return out


def _graphable(op):
    return op is None or getattr(op, "graphable", False)


class _PcgState:
    """Persistent buffers + captured CUDA graphs of one (A, M, n) triple."""

    def __init__(self, apply_A, apply_M, n, host_callables=False):
        torch = __import__("torch")
        self.A, self.M, self.n = apply_A, apply_M, n
        self.host_callables = host_callables
        f64 = dict(dtype=torch.float64, device="cuda")
        self.x, self.r, self.p = (torch.zeros(n, **f64) for _ in range(3))
        self.z, self.Ap = torch.zeros(n, **f64), torch.zeros(n, **f64)
        self.graphs = self.pair = self.loop = None

    def precond(self):
        if self.M is None:
            self.z.copy_(self.r)
        else:
            _apply(self.M, self.r, self.z, self.host_callables)

    def step(self, rz, rz_new, pap=None, rr=None, gate_in=-1, gate_out=-1):
        ws = workspace()
        st = _abi.stream()
        pap = ws.PAP if pap is None else pap
        rr = ws.RR if rr is None else rr
        if hasattr(self.A, "apply_dot") and not _NO_FUSED_PAP:   # p'Ap inside the apply kernel
            self.A.apply_dot(self.p, self.Ap, pap)
        else:
            _apply(self.A, self.p, self.Ap, self.host_callables)
            ws.dot(self.p, self.Ap, pap)
        _abi.call("mcs_cg_update_gated", self.n, _abi.ptr(self.x), _abi.ptr(self.r),
                  _abi.ptr(self.p), _abi.ptr(self.Ap), _abi.ptr(ws.sc), rz, pap, rr, gate_in,
                  gate_out, ws.BNORM, ws.RTOL, _abi.ptr(ws.partials), _abi.ptr(ws.counter), st)
        self.precond()
        ws.dot(self.r, self.z, rz_new)
        _abi.call("mcs_xpby", self.n, _abi.ptr(self.z), _abi.ptr(self.p), _abi.ptr(ws.sc),
                  rz_new, rz, st)

    def capture(self):
        """Record one step per rz-slot parity (the state is restored after
        the eager warm-up the capture needs)."""
        torch = __import__("torch")
        import gc
        ws = workspace()
        saved = [t.clone() for t in (self.x, self.r, self.p, self.z, ws.sc)]
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(cur)
        graphs = []
        # No cyclic garbage collection while a stream is capturing: collecting
        # an older operator's PCG state there destroys its CUDA graphs and
        # frees their private pools (cudaFree / cudaGraphExecDestroy), which
        # invalidates the running capture (seen as error 901 on the next
        # launch).  Pending garbage is collected before the first capture.
        gc_was_enabled = gc.isenabled()
        gc.collect()
        gc.disable()
        try:
            with torch.cuda.stream(side):
                self.step(ws.RZ0, ws.RZ1)
                for rz, rzn in ((ws.RZ0, ws.RZ1), (ws.RZ1, ws.RZ0)):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=side):
                        self.step(rz, rzn)
                    graphs.append(g)
                # two steps per replay: the second is gated off on the device when
                # the first one stops the loop (one host read-back per two steps)
                pair = torch.cuda.CUDAGraph(keep_graph=True)
                with torch.cuda.graph(pair, stream=side):
                    self.step(ws.RZ0, ws.RZ1, gate_out=ws.GATE)
                    self.step(ws.RZ1, ws.RZ0, ws.PAP2, ws.RR2, gate_in=ws.GATE)
                pair.instantiate()
        finally:
            if gc_was_enabled:
                gc.enable()
        cur.wait_stream(side)
        for t, v in zip((self.x, self.r, self.p, self.z, ws.sc), saved):
            t.copy_(v)
        self.graphs = graphs
        self.pair = None if _NO_PAIR else pair
        if self.pair is not None and not _NO_LOOP:
            # the whole loop as one launch: a conditional WHILE node around the
            # pair graph (csrc/pcg_loop.cu)
            import ctypes
            self.hist = torch.zeros(2 + 2 * _LOOP_CAP, dtype=torch.float64, device="cuda")
            out = ctypes.c_void_p()
            _abi.call("mcs_pcg_loop_build", pair.raw_cuda_graph(), _abi.ptr(ws.sc),
                      _abi.ptr(self.hist), ws.PAP, ws.RR, ws.PAP2, ws.RR2, ws.BNORM, ws.RTOL,
                      _LOOP_CAP, ctypes.byref(out))
            self.loop = out.value

    def __del__(self):
        try:
            if getattr(self, "loop", None):
                _abi.call("mcs_pcg_loop_destroy", self.loop)
        except Exception:
            pass


def _state_slot(apply_A):
    """Captured PCG states live on the operator object they were captured
    for (a dict attribute keyed by (id(M), n)), so they are freed together
    with the operator: nothing module-level pins a CondensedSystem, its CUDA
    graphs or their memory pools (the state references the operator back;
    Python's cycle collector reclaims both)."""
    try:
        d = apply_A.__dict__.setdefault("_pcg_states", {})
    except AttributeError:                    # no instance dict: do not cache
        return None
    return d


def release(apply_A, apply_M=None):
    """Drop the captured PCG graphs and buffers of `apply_A` (all
    preconditioners, or only `apply_M`'s) now, instead of at garbage
    collection."""
    d = getattr(apply_A, "__dict__", {}).get("_pcg_states")
    if not d:
        return
    for key in [k for k, st in d.items() if apply_M is None or st.M is apply_M]:
        st = d.pop(key)
        st.__del__()
        st.loop = None
    __import__("gc").collect()
# A/B switch for the fused curvature (MCS_NO_FUSED_PAP=1: separate dot kernel)
_NO_FUSED_PAP = __import__("os").environ.get("MCS_NO_FUSED_PAP", "0") == "1"
# A/B switch for the two-step graph (MCS_NO_PAIR=1: one read-back per step)
_NO_PAIR = __import__("os").environ.get("MCS_NO_PAIR", "0") == "1"
# A/B switch for the single-launch loop (MCS_NO_LOOP=1: one launch per pair)
_NO_LOOP = __import__("os").environ.get("MCS_NO_LOOP", "0") == "1"
_LOOP_CAP = 4096   # steps of device-side (p'Ap, rr) history


@_abi.nvtx("cg")
def cg(apply_A, b, apply_M=None, rtol=1e-8, maxit=1000, stream=None, use_graph=True):
    """Preconditioned CG.  `apply_A` / `apply_M` are device operators
    (objects with `.apply(v, out=)`, or callables on CUDA tensors).  `b` may
    be NumPy (returns NumPy) or a CUDA tensor (returns a CUDA tensor).

    When both operators are this package's device operators, one PCG step
    (A p, p'Ap, the x/r update with ||r||^2, z = M r, r'z, the p update) is
    captured into CUDA graphs (once per operator pair, cached).  The main
    graph holds TWO steps: the first one's x/r update kernel evaluates the
    host's stopping test (negative curvature, or sqrt(rr)/bnorm <= rtol,
    same IEEE operations) into a device gate, and the second step's update
    is a no-op when the gate is set, so one graph launch and one read-back
    serve two iterations (single-step graphs per rz parity finish an odd
    maxit).  A step computes z = M r before the host has seen the stopping
    test; when the test stops the loop that z is unused, so x, the residual
    history and the iteration count are the reference loop's.  By default the
    pairs themselves run inside ONE launch: a conditional WHILE graph node
    around the pair graph, with a record kernel that appends each step's
    (p'Ap, rr) to a device history and applies the same stopping test
    (csrc/pcg_loop.cu); the host reads the history once per solve."""
    import os
    bd, host = as_device(b)
    n = bd.numel()
    ws: Workspace = workspace()
    sc = ws.sc
    # MCS_NO_GRAPH=1: eager launches (ncu launch lists; ncu does not replay graphs)
    use_graph = use_graph and os.environ.get("MCS_NO_GRAPH", "0") != "1"
    graphable = use_graph and _graphable(apply_A) and _graphable(apply_M)
    slots = _state_slot(apply_A) if graphable else None
    key = (id(apply_M), n)
    S = slots.get(key) if slots is not None else None
    if S is None or S.A is not apply_A or S.M is not apply_M:
        S = _PcgState(apply_A, apply_M, n, host_callables=host)
        if slots is not None:
            slots[key] = S
    S.x.zero_()
    S.r.copy_(bd)
    ws.dot(bd, bd, ws.BB)
    bb = float(sc[ws.BB].item())
    report = KrylovReport(residuals=[1.0])
    if bb == 0.0:
        report.converged = True
        x = S.x.clone()
        return (x.cpu().numpy() if host else x), report
    bnorm = np.sqrt(bb)
    S.precond()
    S.p.copy_(S.z)
    ws.dot(S.r, S.z, ws.RZ0)
    if graphable and S.graphs is None and maxit > 2:
        S.capture()
    rz, rz_new = ws.RZ0, ws.RZ1
    sc[ws.BNORM] = bnorm
    sc[ws.RTOL] = rtol
    it = 0

    def record(pap, rr):
        """The reference loop's per-step control flow; True = stop.  The
        device gates (blas1.cu cg_update_kernel, pcg_loop.cu) use the same
        predicates: pAp <= 0 raises, res <= rtol stops, and a NaN passes
        both (the reference then runs on to maxit, not converged)."""
        if pap <= 0:
            raise NegativeCurvatureError(f"p'Ap = {pap:.3e} at iteration {it}")
        res = float(np.sqrt(rr) / bnorm)
        report.residuals.append(res)
        report.iterations = it
        report.converged = res <= rtol
        return report.converged

    if S.loop is not None and maxit >= 2:
        # one launch runs pairs until the device-side test stops; the host
        # replays the same test over the recorded (p'Ap, rr) history
        _abi.call("mcs_pcg_loop_launch", S.loop, _abi.ptr(S.hist), min(maxit, _LOOP_CAP),
                  _abi.stream())
        ns = int(S.hist[0].item())
        v = S.hist[2:2 + 2 * ns].tolist()
        for q in range(ns):
            it += 1
            if record(v[2 * q], v[2 * q + 1]):
                break
            rz, rz_new = rz_new, rz
    while it < maxit and not report.converged:
        if S.pair is not None and rz == ws.RZ0 and it + 2 <= maxit:
            S.pair.replay()
            v = sc[ws.PAP:ws.RR2 + 1].tolist()
            steps = ((v[0], v[1]), (v[ws.PAP2 - ws.PAP], v[ws.RR2 - ws.PAP]))
        else:
            if S.graphs is not None:
                S.graphs[0 if rz == ws.RZ0 else 1].replay()
            else:
                S.step(rz, rz_new)
            steps = (tuple(sc[ws.PAP:ws.RR + 1].tolist()),)
        for pap, rr in steps:
            it += 1
            if record(pap, rr):
                break
            rz, rz_new = rz_new, rz
    x = S.x.clone()
    return (x.cpu().numpy() if host else x), report


def _norm(ws: Workspace, v) -> float:
    ws.dot(v, v, ws.TMP)
    return float(np.sqrt(ws.sc[ws.TMP].item()))


def _op(op, v, out, host_callables=False):
    return _apply(op, v, out, host_callables)


# MCS_GS_FUSED=1: the fused second-pass kernel (one basis read for w - V h1,
# V^T w' and ||w'||; three basis reads per step instead of four).  Measured
# slower at cfg2 (727 vs 365 ms for 246 steps, profiles/r02/gmres_gs_fused.txt):
# each CTA's tile sweep serialises load -> products -> barriers, and the
# plain multi-dot / GEMV kernels already run near the HBM rate.
_GS_FUSED = __import__("os").environ.get("MCS_GS_FUSED", "0") == "1"
# Gram-Schmidt accounting of `gmres` (diagnostics: tools/gmres_prof.py)
_GS_STATS = {"steps": 0, "second_pass": 0}


@_abi.nvtx("gmres")
def gmres(apply_A, b, apply_M=None, rtol=1e-6, maxit=500, project=None, x0=None):
    """Full (non-restarted) right-preconditioned GMRES (reference
    `krylov.py:25-100`) with the Krylov basis in HBM.

    Same control flow and reporting as the reference: optional null-space
    `project` on b and on every new direction, residual history of the
    Givens-rotated least-squares residual, happy-breakdown test
    h_{j+1,j} <= 1e-14 |rotated diagonal|, FloatingPointError on a
    non-finite h, x = x0 + M (V y).  The Arnoldi orthogonalisation is
    classical Gram-Schmidt with DGKS re-orthogonalisation (one or two
    deterministic V w / V^T h product pairs per step, csrc/stokes.cu)
    instead of the reference's modified Gram-Schmidt loop: the same
    Hessenberg matrix up to rounding, with one host read-back of the column
    per step.  The small
    (maxit+1) x maxit least-squares problem stays on the host, as in the
    reference."""
    import torch
    bd, host = as_device(b)
    ws: Workspace = workspace()
    n = bd.numel()
    ident = apply_M is None
    b_ = bd.clone()
    if project is not None:
        b_ = project(b_)
    x0d = torch.zeros(n, dtype=torch.float64, device="cuda") if x0 is None else as_device(x0)[0]
    if x0 is not None and _norm(ws, x0d) > 0.0:
        r0 = b_ - _op(apply_A, x0d, empty(n), host)
    else:
        r0 = b_.clone()
    beta = _norm(ws, r0)
    bnorm = _norm(ws, b_)
    report = KrylovReport(residuals=[1.0 if bnorm == 0 else beta / bnorm])

    def finish(x):
        x = x if host is False else x.cpu().numpy()
        return x, report

    if bnorm == 0.0 or beta / bnorm <= rtol:
        report.converged = True
        return finish(x0d)
    cap = min(maxit + 1, 64)
    V = torch.empty((cap, n), dtype=torch.float64, device="cuda")
    _abi.call("mcs_axpby", n, 1.0 / beta, _abi.ptr(r0), 0.0, _abi.ptr(V[0]), _abi.stream(None))
    H = np.zeros((maxit + 1, maxit))
    cs, sn = np.zeros(maxit), np.zeros(maxit)
    g = np.zeros(maxit + 1)
    g[0] = beta
    partial = torch.empty(_abi.call("mcs_mdot_len") * (maxit + 1), dtype=torch.float64,
                          device="cuda")
    # the per-step read-back (||w|| before / after each pass, gate, both h
    # columns): two D2H copies into one pinned buffer, no gather kernel
    # fused second-pass products (one basis read for w - V h1, V^T w' and ||w'||)
    nblk = _abi.call("mcs_gs_fused_blocks")
    ph2 = torch.empty((maxit + 1) * nblk, dtype=torch.float64, device="cuda")
    pnrm = torch.empty(nblk, dtype=torch.float64, device="cuda")
    hh = torch.empty(2 * (maxit + 1), dtype=torch.float64, device="cuda")
    h1, h2 = hh[:maxit + 1], hh[maxit + 1:]
    nsc = ws.TMP3 - ws.TMP + 1
    back_h = torch.empty(nsc + 2 * (maxit + 1), dtype=torch.float64).pin_memory()
    z, w = empty(n), empty(n)
    j = 0
    while j < maxit:
        mz = V[j] if ident else _op(apply_M, V[j], z, host)
        _op(apply_A, mz, w, host)
        if project is not None:
            w = project(w)
        m = j + 1
        # classical Gram-Schmidt, repeated once when the first pass lost more
        # than half the norm (DGKS criterion 1/sqrt(2)): MGS-quality
        # orthogonality at the cost of one or two V w / V^T h pairs per step.
        # ||w|| before and after the pass and the h column come back in ONE
        # read-back (a second one only when the second pass runs).
        ws.dot(w, w, ws.TMP)
        _abi.call("mcs_mdot", m, n, n, _abi.ptr(V), _abi.ptr(w), _abi.ptr(partial),
                  _abi.ptr(h1), _abi.stream(None))
        # the DGKS decision on the device: the second pass is launched always
        # and skipped by its kernels when the first one kept enough of ||w||
        gate = ws.sc.data_ptr() + 8 * ws.GS_GATE
        rc = -1000
        if _GS_FUSED:   # w -= V h1, h2 = V^T w, ||w||^2 and the gate from one basis read
            rc = _abi.lib().mcs_gs_fused(
                m, n, n, _abi.ptr(V), _abi.ptr(w), _abi.ptr(h1), _abi.ptr(ph2), _abi.ptr(pnrm),
                _abi.ptr(h2), _abi.ptr(ws.sc), ws.TMP, ws.TMP2, ws.GS_GATE, _abi.stream(None))
            if rc not in (0, -1000):
                raise _abi.McsError(f"mcs_gs_fused failed with CUDA error {-rc}")
        if rc != 0:     # the default; also m beyond the fused kernel's shared-memory tile
            _abi.call("mcs_gemv_acc", m, n, n, _abi.ptr(V), _abi.ptr(h1), -1.0, 1.0,
                      _abi.ptr(w), _abi.stream(None))
            ws.dot(w, w, ws.TMP2)
            _abi.call("mcs_gs_gate", _abi.ptr(ws.sc), ws.TMP, ws.TMP2, ws.GS_GATE,
                      _abi.stream(None))
            _abi.call("mcs_mdot_gated", m, n, n, _abi.ptr(V), _abi.ptr(w), _abi.ptr(partial),
                      _abi.ptr(h2), gate, _abi.stream(None))
        _abi.call("mcs_gemv_acc_gated", m, n, n, _abi.ptr(V), _abi.ptr(h2), -1.0, 1.0,
                  _abi.ptr(w), gate, _abi.stream(None))
        ws.dot(w, w, ws.TMP3)
        back_h[:nsc].copy_(ws.sc[ws.TMP:ws.TMP3 + 1], non_blocking=True)
        back_h[nsc:nsc + m].copy_(h1[:m], non_blocking=True)
        back_h[nsc + m:nsc + 2 * m].copy_(h2[:m], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        back = back_h.numpy()
        wnorm, hnext = float(np.sqrt(back[0])), float(np.sqrt(back[ws.TMP2 - ws.TMP]))
        o = nsc
        hcol = back[o:o + m].copy()
        _GS_STATS["steps"] += 1
        second = not hnext > 0.7071067811865476 * wnorm
        if second != (back[ws.GS_GATE - ws.TMP] == 0.0):
            raise RuntimeError("device and host Gram-Schmidt decisions differ")
        if second:
            _GS_STATS["second_pass"] += 1
            hnext = float(np.sqrt(back[ws.TMP3 - ws.TMP]))
            hcol = hcol + back[o + m:o + 2 * m]
        H[:m, j] = hcol
        H[j + 1, j] = hnext
        if not np.isfinite(hnext) or not np.all(np.isfinite(hcol)):
            raise FloatingPointError("GMRES residual became non-finite")
        for i in range(j):                                # accumulated Givens rotations
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        hsub = H[j + 1, j]
        denom = np.hypot(H[j, j], hsub)
        cs[j] = H[j, j] / denom
        sn[j] = hsub / denom
        H[j, j] = denom
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        res = abs(g[j + 1]) / bnorm
        report.residuals.append(res)
        happy = hsub <= 1e-14 * denom
        if not happy:
            if j + 1 >= V.shape[0]:                       # grow the basis
                Vn = torch.empty((min(maxit + 1, 2 * V.shape[0]), n), dtype=torch.float64,
                                 device="cuda")
                Vn[:V.shape[0]].copy_(V)
                V = Vn
            _abi.call("mcs_axpby", n, 1.0 / hsub, _abi.ptr(w), 0.0, _abi.ptr(V[j + 1]),
                      _abi.stream(None))           # V[j+1] = w / h_{j+1,j}, one kernel
        j += 1
        if res <= rtol or happy:
            report.converged = True
            break
    mm = j
    y = np.linalg.solve(H[:mm, :mm], g[:mm])
    yd = torch.from_numpy(y).cuda()
    t = empty(n)
    _abi.call("mcs_gemv_acc", mm, n, n, _abi.ptr(V), _abi.ptr(yd), 1.0, 0.0, _abi.ptr(t), _abi.stream(None))
    xk = x0d + (t if ident else _op(apply_M, t, empty(n), host))
    if project is not None:
        xk = project(xk)
    report.iterations = mm
    return finish(xk)
