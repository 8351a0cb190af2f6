#!/usr/bin/env python
"""Benchmark of the B200 condensation + PCG hot path (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (BASELINE.json configs[1]): N=128 grid, 32,768
jittered triangles, k=4, nu=1e-2, Fourier body force seed 0.  One *step* is
one condensation pass over all elements on the GPU: element blocks from the
geometry (A1) -> sigma/omega elimination (A3) -> double Schur (A4), one
fused kernel at k <= 4.  `value` = elements condensed per second, inputs
resident in HBM, L2 flushed before every timed step, device time by CUDA
events; `roofline` reports the kernel against the measured FP64 peak with
SURVEY §8.0.1's algorithmic flops (executed flops alongside).

The same run measures, at cfg2 and again at the largest config (cfg3: N=256,
131,072 triangles, k=6, the `cfg3` block): the condensed-operator apply
(DOF/s, % HBM), the facet Jacobi (% HBM), the full PCG solve to rtol 1e-8 for
both compositions with its iteration count checked against the reference's
(tests/golden/cfg{2,3}_full.npz, produced by running the reference;
|delta| > 1 aborts the bench) and the time against the §8.0.1 HBM-bound PCG;
the config-5 SPD-Schur microbench; the Stokes-mode GMRES; `e2e` through the
C ABI with host buffers; and on rank 0 the CPU baselines: the reference
condensation algorithm (oracle port, `cpu_baseline`) and the reference's
CPU solver path on the same matrices (`cpu_solver_baselines`).

`--impl reference` times the reference algorithm's CPU restatement
(oracle/mcs_oracle.py: quadrature blocks + LU condensation + double Schur,
condensation.py:159-224 / assembly.py:49-91) on all host cores, process
parallel over elements, one step = every element of the workload.

Multi-GPU (torchrun, N>1): replicas only - every rank condenses
its own copy of the workload; value = all ranks' elements / max-over-ranks
time.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("elements condensed/s and condensed-apply DOF/s at 1 GPU; "
          "% FP64/HBM roofline")
WORKLOAD = ("cfg2: unit square N=128 (32,768 triangles, jitter 0.2h seed 1), k=4, "
            "nu=1e-2, Fourier force seed 0; step = A1 element blocks + A3 "
            "sigma/omega condensation + A4 double Schur over all elements")


def flops_per_element(k):
    z = dict(ns=3 * (k + 1) * (k + 2) // 2 - 3, nw=k * (k + 1) // 2,
             nloc=(k + 1) * (k + 2) + 3 * k, nint=(k + 1) * (k - 1))
    ns, nw, nl, ni = z["ns"], z["nw"], z["nloc"], z["nint"]
    nc = nl - ni
    f_cond = (ns ** 3 / 3 + ns ** 2 * (nl + nw) + nw ** 2 * ns + nw ** 3 / 3
              + 2 * nw * ns * nl + nw ** 2 * nl + nl ** 2 * ns + nl ** 2 * nw)
    f_ds = ni ** 3 / 3 + ni ** 2 * nc + nc ** 2 * ni
    return f_cond, f_ds


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
                power.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# -------------------------------------------------------------- our arm

def load_peaks():
    peaks = {"hbm_gbs": None, "fp64_tflops": None}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks["hbm_gbs"] = json.load(fh).get("hbm_gbs")
    except OSError:
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")) as fh:
            d = json.load(fh)
            peaks["fp64_tflops"] = max(d["dfma_tflops"], d["dmma_m8n8k4_tflops"])
    except OSError:
        pass
    if peaks["hbm_gbs"] is None:
        peaks["hbm_gbs"] = 6650.0
    return peaks


def ncu_traffic(prefix):
    """DRAM bytes (read + write) per launch of the kernel whose name starts
    with `prefix`, from the newest committed `ncu --set full` summary
    (profiles/ncu_kernels_*.json) that has it."""
    import glob
    paths = glob.glob(os.path.join(ROOT, "profiles", "ncu_kernels_*.json")) + \
        glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_kernels_*.json"))
    # newest round first (the round directory / file suffix), then mtime
    for path in sorted(paths, key=lambda p_: (os.path.basename(os.path.dirname(p_)), p_),
                       reverse=True):
        try:
            with open(path) as fh:
                d = json.load(fh)
        except (OSError, ValueError):
            continue
        for name, rec in d.items():
            if name.startswith(prefix):
                return rec.get("dram_bytes")
    return None


def flops_structured(k):
    """FP64 flops per element of the structured path actually executed
    (DESIGN.md §5): Bsig generation, block factors, Y, S_T = adiv + Y Y^T,
    and the double Schur (Cholesky, L^-1, W = L^-1 S_oc, X = L^-T W,
    S_oo^-1 = L^-T L^-1, Sd = S_cc - W^T W).  2 flops per FMA."""
    ns = 3 * (k + 1) * (k + 2) // 2 - 3
    nu, nh = (k + 1) * (k + 2), 3 * k
    nl_, ni = nu + nh, (k + 1) * (k - 1)
    nc, nem = nl_ - ni, 3 * (k + 1)
    ml, nb = k * (k + 1) // 2, 3 * k
    ny = 2 * ml + nb
    gen = 2 * 3 * ns * (nem + nh)
    fac = 2 * 6 * nb * nb + 2 * nb ** 3 / 3 + ml * (2 * 6 * 9 + 60)
    y = nl_ * (2 * 6 * ml + nb * (nb + 1))
    syrk = nl_ * (nl_ + 1) * ny + nu * (nu + 1)
    ds = ni ** 3 + 2 * ni * ni * nc + nc * (nc + 1) * ni
    return gen + fac + y + syrk + ds


def max_over_ranks(x: float, world: int, device) -> float:
    """Whole-job time of N replicas: the maximum over ranks (all_reduce MAX on
    the process group's device; identity for one rank)."""
    if world <= 1:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def _golden(name):
    """Reference-generated fixture (tests/golden, oracle/make_golden_full.py)
    or None.  Read for its iteration counts / vectors only: the bench never
    touches /root/reference."""
    path = os.path.join(ROOT, "tests", "golden", name + ".npz")
    return np.load(path) if os.path.exists(path) else None


def _rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _vec_parity(got, g, key):
    """Relative l2 error of a solver vector against a golden one (full vector,
    or the fixture's seeded sample for cfg3)."""
    if g is None:
        return None
    got = np.asarray(got)
    if key in g:
        return _rel(got, g[key])
    if key + "_sample" in g:
        return _rel(got[g["sample_idx"]], g[key + "_sample"])
    return None


def pcg_hbm_bytes(sys_, M, comp):
    """SURVEY §8.0.1 algorithmic HBM bytes of one PCG iteration:
    B_apply + B_ext + B_jac + B_E + B_coarse + B_vec (+ 2 S_d applies for
    the multiplicative composition)."""
    z = sys_.z
    nt = sys_.S_dev.shape[0]
    nl, ni, nc = z["nloc"], z["n_int"], z["ncpl"]
    nv, ncf = sys_.maps.n_vv_free, sys_.maps.n_cpl_free
    asp = M.inner
    sm = asp.smoother
    b = 2 * sys_.k + 1
    B = {"apply": nt * 8 * nl * (nl + 1) / 2 + 16 * nv,
         "ext": nt * 8 * (ni * (ni + 1) / 2 + 2 * ni * nc),
         "jacobi": sm.nblk * 8 * b * (b + 1) / 2 + 16 * ncf,
         "vec": 10 * 8 * nv}
    nnzE = int(asp.E.val.numel())
    ncoarse = asp.coarse.n
    B["embedding"] = 2 * (nnzE * 12 + 8 * 2 * (ncf + ncoarse))
    F = asp.coarse.data
    if asp.coarse.kind == "dense":
        nnzL = ncoarse * (ncoarse + 1) // 2
    else:
        nnzL = sum(len(nd.own) * (len(nd.own) + 1) // 2 + len(nd.own) * len(nd.B)
                   for nd in F.nodes)
    B["coarse"] = 2 * nnzL * 12
    if comp == "multiplicative":
        B["sd_applies"] = 2 * (nt * 8 * nc * (nc + 1) / 2 + 16 * ncf)
    return B


def run_config(args, cfg, dev, world, steps, warmup, l2_flush, peaks, full=True):
    """One BASELINE config on the GPU: condensation (timed `steps` times,
    L2 flushed before each), then S apply, facet Jacobi and PCG (both
    compositions) with parity against the reference fixtures."""
    import torch
    from paper_2207_08481_b200 import _abi, engine, refblocks
    from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur
    from paper_2207_08481_b200.dofmap import FeSystem
    from paper_2207_08481_b200.driver import (SolverOptions, condensed_rhs,
                                               velocity_preconditioner)
    from paper_2207_08481_b200.krylov import cg, release
    from paper_2207_08481_b200.operators import SOperator
    from paper_2207_08481_b200.problems import baseline_config

    prob = baseline_config(cfg, args.n)
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    k, nt = prob.k, prob.mesh.num_triangles
    z = refblocks.local_sizes(k)
    refs = refblocks.build_refs(fes)
    W_h = refblocks.element_weights(fes, prob.nu)
    W = engine.to_dev(W_h)
    ST = torch.empty((nt, engine.st_stride(k)), dtype=torch.float64, device=dev)
    ext = torch.empty((nt, _abi.call("mcs_ext_stride", k)), dtype=torch.float64, device=dev)
    Sd = torch.empty((nt, _abi.call("mcs_sd_stride", k)), dtype=torch.float64, device=dev)
    info = torch.empty(nt, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    st = _abi.stream(stream)
    fused = k in engine.FUSED_DEGREES
    tab = engine.to_dev(engine.fused_tables(refs)[0])

    def launch(a, b, ev=None):
        """The condensation of elements [a, b): A1 + A3 + A4.  k <= 4: one
        warp-per-element kernel; k = 5, 6: the generation-fused condensation
        pipeline in passes (mcs_condense_gen), then the register-resident
        warp-per-element double Schur (the library defaults)."""
        if fused:
            _abi.call("mcs_condense_fused", k, b - a, _abi.ptr(W[a:b]), W.shape[1],
                      _abi.ptr(tab), _abi.ptr(ST[a:b]), _abi.ptr(ext[a:b]),
                      _abi.ptr(Sd[a:b]), _abi.ptr(info[a:b]), st)
            if ev:
                ev.record(stream)
            return 1
        _abi.call("mcs_condense_gen", k, b - a, _abi.ptr(W[a:b]), W.shape[1], _abi.ptr(tab),
                  _abi.ptr(ST[a:b]), _abi.ptr(info[a:b]), st)
        if ev:
            ev.record(stream)
        _abi.call("mcs_double_schur", k, b - a, _abi.ptr(ST[a:b]), _abi.ptr(ext[a:b]),
                  _abi.ptr(Sd[a:b]), _abi.ptr(info[a:b]), st)
        return 3      # lane-table kernel + condensation + double Schur

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        n = launch(0, nt, ev[1] if ev else None)
        if ev:
            ev[2].record(stream)
        return n

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if int(info.abs().sum().item()):
        raise RuntimeError("condensation reported failing elements")
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    launches = 0
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    for i in range(steps):
        l2_flush(i)                    # untimed: 256 MiB write + 256 MiB read
        launches += step(evs[i])
    torch.cuda.synchronize()
    t_step = np.array([e[0].elapsed_time(e[2]) for e in evs])
    t_first = np.array([e[0].elapsed_time(e[1]) for e in evs])
    ms_per_step = max_over_ranks(float(t_step.mean()), world, dev)
    f_cond, f_ds = flops_per_element(k)
    f_alg = f_cond + f_ds
    f_exec = flops_structured(k)
    out = {"elements": nt, "k": k, "ms": ms_per_step,
           "elements_per_s": world * nt / (ms_per_step * 1e-3), "gpu_launches": launches}
    if fused:
        out["breakdown_ms"] = {"condense_fused (A1+A3+A4, one kernel)": float(t_step.mean())}
        kname, kpref, t_kern = (f"condense_fused (A1+A3+A4), k={k}",
                                f"condense_fused_kernel<{k},", float(t_step.mean()))
        f_kern_alg, f_kern_exec = f_alg, f_exec
    else:
        t_a3 = float(t_first.mean())
        out["breakdown_ms"] = {"condense_fused passes (A1+A3)": t_a3,
                               "double_schur_reg (A4)": float((t_step - t_first).mean())}
        kname, kpref, t_kern = (f"condense_fused passes (A1+A3), k={k}",
                                f"condense_fused_kernel<{k},", t_a3)
        f_kern_alg = f_cond
        z_ = z
        ny_ = k * (k + 1) + 3 * k
        f_kern_exec = (z_["nloc"] * (z_["nloc"] + 1) * ny_ + z_["nloc"] * (
            12 * (k * (k + 1) // 2) + 3 * k * (3 * k + 1)))
    P = peaks["fp64_tflops"]
    ach = f_kern_alg * nt / (t_kern * 1e-3) / 1e12
    step_ach = f_alg * nt / (ms_per_step * 1e-3) / 1e12
    out["roofline"] = {
        "bound": "tensor", "pipe": "FP64 tensor cores (DMMA m8n8k4) + FP64 FMA",
        "kernel": kname, "achieved": ach, "peak": P, "unit": "TFLOP/s", "frac": ach / P,
        "flops_per_element": f_kern_alg,
        "flops_definition": "SURVEY §8.0.1 algorithmic: F_cond" + (" + F_ds" if fused else "")
                            + " per element (dense two-stage Cholesky formulation); "
                            "step_achieved uses F_cond + F_ds over the whole step",
        "executed_flops_per_element": f_kern_exec,
        "executed_tflops": f_kern_exec * nt / (t_kern * 1e-3) / 1e12,
        "executed_frac": f_kern_exec * nt / (t_kern * 1e-3) / 1e12 / P,
        "step_achieved": step_ach, "step_frac": step_ach / P,
        "traffic": ncu_traffic(kpref),
        "note": "frac counts the dense formulation's flops (SURVEY §8.0.1), so the structured "
                "algebra (DESIGN.md §3.2, ~2.5x fewer flops at k = 4, ~4x at k = 6) can exceed 1; "
                "executed_frac counts the flops the kernels issue",
        "peak_source": "profiles/fp64_peak_r01.json (measured DMMA m8n8k4 peak, B200)"}
    res = {"condensation": out, "_step": step, "_launch": launch,
           "_bufs": (W, W_h, ST, ext, Sd, info, fused), "prob": prob}
    if not full:
        return res

    # ---- condensed-operator apply (A6), facet Jacobi (A9), PCG (A8-A13)
    g = _golden(f"cfg{cfg}_full") if not args.n else None
    sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
    S = SOperator(sys_)
    n_free = sys_.maps.n_vv_free
    x = torch.randn(n_free, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    for _ in range(5):
        S.apply(x, out=y)
    napp = max(20, steps)
    ev_a = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(napp)]
    for i in range(napp):
        l2_flush(i)
        ev_a[i][0].record(stream)
        S.apply(x, out=y)
        ev_a[i][1].record(stream)
    torch.cuda.synchronize()
    t_apply = float(np.mean([e[0].elapsed_time(e[1]) for e in ev_a]))
    apply_bytes = nt * 8 * z["nloc"] * (z["nloc"] + 1) / 2 + 16 * n_free
    hbm = peaks["hbm_gbs"]
    res["apply"] = {"dof_per_s": n_free / (t_apply * 1e-3), "ms": t_apply, "n_vv_free": n_free,
                    "roofline": {"bound": "hbm", "achieved": apply_bytes / (t_apply * 1e-3) / 1e9,
                                 "peak": hbm, "unit": "GB/s",
                                 "frac": apply_bytes / (t_apply * 1e-3) / 1e9 / hbm,
                                 "algorithmic_bytes": apply_bytes,
                                 "traffic": ncu_traffic(f"elem_apply_kernel<{z['nloc']},")}}
    if g is not None:
        v = np.random.default_rng(11).standard_normal(n_free)
        res["apply"]["parity_rel_l2_vs_reference"] = _vec_parity(S(v), g, "probe_Sv")
    pcg = {}
    for comp in ("additive", "multiplicative"):
        t0 = time.perf_counter()
        M = velocity_preconditioner(fes, sys_, prob.nu,
                                    SolverOptions(smoother="jacobi", composition=comp))
        torch.cuda.synchronize()
        t_sup = time.perf_counter() - t0
        if "jacobi" not in res:
            sm = M.inner.smoother
            nc = sys_.maps.n_cpl_free
            rj = torch.randn(nc, dtype=torch.float64, device=dev)
            xj = torch.empty_like(rj)
            for _ in range(5):
                sm.jacobi_apply(rj, out=xj)
            ev_j = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(napp)]
            for i in range(napp):
                l2_flush(i)
                ev_j[i][0].record(stream)
                sm.jacobi_apply(rj, out=xj)
                ev_j[i][1].record(stream)
            torch.cuda.synchronize()
            t_jac = float(np.mean([e[0].elapsed_time(e[1]) for e in ev_j]))
            bsz = 2 * k + 1
            jac_bytes = sm.nblk * 8 * bsz * (bsz + 1) / 2 + 16 * nc
            res["jacobi"] = {"kernel": f"jacobi_apply_kernel<{bsz}>", "ms": t_jac,
                             "bound": "hbm", "achieved": jac_bytes / (t_jac * 1e-3) / 1e9,
                             "peak": hbm, "unit": "GB/s",
                             "frac": jac_bytes / (t_jac * 1e-3) / 1e9 / hbm,
                             "algorithmic_bytes": jac_bytes,
                             "note": "event time, L2 flushed, launch latency included"}
        b_h = condensed_rhs(fes, sys_)[0]
        b = torch.from_numpy(b_h).to(dev)
        cg(S, b, M, rtol=1e-8, maxit=2000)       # warm-up (captures the CUDA graphs)
        torch.cuda.synchronize()
        solves = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            xs, rep = cg(S, b, M, rtol=1e-8, maxit=2000)
            e1.record(stream)
            torch.cuda.synchronize()
            solves.append(e0.elapsed_time(e1))
        solve_ms = float(np.median(solves))
        Bit = pcg_hbm_bytes(sys_, M, comp)
        bound_ms = rep.iterations * sum(Bit.values()) / (hbm * 1e9) * 1e3
        ref_it = int(g[f"cg_{comp}_iters"]) if g is not None else None
        pcg[comp] = {"iterations": rep.iterations, "final_res": rep.residuals[-1],
                     "solve_ms": solve_ms, "ms_per_iteration": solve_ms / rep.iterations,
                     "precond_setup_s": round(t_sup, 3), "jacobi_scale": M.inner.jacobi_scale,
                     "reference_iterations": ref_it,
                     "iterations_within_1": None if ref_it is None
                     else abs(rep.iterations - ref_it) <= 1,
                     "x_rel_l2_vs_reference": _vec_parity(xs.cpu().numpy(), g, f"cg_{comp}_x"),
                     "hbm_bound_ms": bound_ms, "frac_of_hbm_bound_pcg": bound_ms / solve_ms,
                     "hbm_bytes_per_iteration": {a: float(v) for a, v in Bit.items()}}
        if ref_it is not None and abs(rep.iterations - ref_it) > 1:
            raise RuntimeError(f"cfg{cfg} {comp}: {rep.iterations} PCG iterations, "
                               f"reference {ref_it}")
        if comp == "additive":
            res["_M_add"] = M
        else:
            release(S, M)
    res["pcg"] = pcg
    res["_sys"], res["_S"] = sys_, S
    return res


def run_ours(args, rank, world):
    import torch
    from paper_2207_08481_b200 import _abi

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    _abi.lib()
    flush = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device=dev)
    # after the 256 MiB write, a 256 MiB read of a second buffer evicts the
    # write's dirty lines, so their write-back is not charged to the timed
    # kernel (tools/read_bw_probe.cu: a 256 MB read runs at 4.3 TB/s behind
    # a dirty L2 and 5.6 TB/s behind a clean one)
    flush_rd = torch.ones(256 * 2 ** 20 // 8, dtype=torch.float64, device=dev)

    def l2_flush(i):
        flush.fill_(float(i))
        return flush_rd.sum()

    stream = torch.cuda.current_stream()
    peaks = load_peaks()
    clocks = ClockSampler(dev.index)
    clocks.start()
    time.sleep(0.2)
    head = run_config(args, args.cfg, dev, world, args.steps, args.warmup, l2_flush, peaks)
    clk = clocks.stop()
    cond = head["condensation"]
    W, W_h, ST, ext, Sd_, info, fused = head["_bufs"]
    nt = cond["elements"]

    # ---- e2e through the C ABI with host buffers: H2D weights, D2H results
    W_pin = torch.from_numpy(W_h).pin_memory()
    out_bytes = (ST.numel() + Sd_.numel() + ext.numel()) * 8
    ST_h = torch.empty(ST.shape, dtype=torch.float64).pin_memory()
    Sd_h = torch.empty(Sd_.shape, dtype=torch.float64).pin_memory()
    ext_h = torch.empty(ext.shape, dtype=torch.float64).pin_memory()
    e2e_times = []
    # the elements go through in chunks; chunk c's results leave for the
    # host on a copy stream (its own DMA engine) while chunk c+1 is condensed
    nch = args.e2e_chunks
    chk = [0, nt // 3, nt // 2, nt - 1]
    ref_rows = [t[chk].cpu() for t in (ST, ext, Sd_)]   # from the full-grid launches above
    bounds = [nt * c // nch for c in range(nch + 1)]
    d2h = torch.cuda.Stream()
    done = [torch.cuda.Event() for _ in range(nch)]

    def e2e_step():
        for c in range(nch):
            a, b = bounds[c], bounds[c + 1]
            W[a:b].copy_(W_pin[a:b], non_blocking=True)
            head["_launch"](a, b)
            done[c].record(stream)
            d2h.wait_event(done[c])
            with torch.cuda.stream(d2h):
                ST_h[a:b].copy_(ST[a:b], non_blocking=True)
                Sd_h[a:b].copy_(Sd_[a:b], non_blocking=True)
                ext_h[a:b].copy_(ext[a:b], non_blocking=True)
        stream.wait_stream(d2h)

    for i in range(max(3, min(args.steps, 20)) + 2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            e2e_times.append(e0.elapsed_time(e1))
    e2e_ms = max_over_ranks(float(np.mean(e2e_times)), world, dev)   # the slowest replica
    if int(info.abs().sum().item()):
        raise RuntimeError("e2e condensation reported failing elements")
    if not all(torch.equal(h[chk], r) for h, r in zip((ST_h, ext_h, Sd_h), ref_rows)):
        raise RuntimeError("e2e host buffers differ from the device results")

    # ---- e2e of the PCG solve through the public API: rhs from host, x to host
    from paper_2207_08481_b200.krylov import cg
    b_pin = torch.from_numpy(np.ascontiguousarray(
        __import__("paper_2207_08481_b200.driver", fromlist=["condensed_rhs"]).condensed_rhs(
            head["_sys"].fes, head["_sys"])[0])).pin_memory()
    x_pin = torch.empty_like(b_pin).pin_memory()
    bd = torch.empty(b_pin.shape, dtype=torch.float64, device=dev)
    pcg_e2e = []
    for i in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        bd.copy_(b_pin, non_blocking=True)
        xs, rep = cg(head["_S"], bd, head["_M_add"], rtol=1e-8, maxit=2000)
        x_pin.copy_(xs, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 1:
            pcg_e2e.append(e0.elapsed_time(e1))

    # ---- config-5 microbench (SPD Schur S = B^T A^-1 B, n_s=60, n_c=36)
    micro = run_microbench(args, dev) if args.micro else None
    stokes = run_stokes(head["_sys"].fes, head["_sys"], head["prob"], dev) if args.stokes else None
    cpu_extra = cpu_solver_baselines(head) if (rank == 0 and args.cpu_solver) else None
    for key in ("_M_add", "_S", "_sys", "_bufs", "_step", "_launch"):
        head.pop(key, None)

    # ---- the largest BASELINE config (cfg3, k = 6) in the same run
    big = None
    if args.cfg3 and args.cfg == 2 and not args.n:
        torch.cuda.empty_cache()
        clk3 = ClockSampler(dev.index)
        clk3.start()
        time.sleep(0.1)
        big = run_config(args, 3, dev, world, max(3, min(args.steps, 10)), 3, l2_flush, peaks)
        big["clocks"] = clk3.stop()
        for key in ("_M_add", "_S", "_sys", "_bufs", "_step", "_launch", "prob"):
            big.pop(key, None)

    out = {
        "metric": METRIC, "value": cond["elements_per_s"], "unit": "elements/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cond["ms"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded SURVEY §8d generators)",
        "config": {"workload": WORKLOAD if args.cfg == 2 else f"cfg{args.cfg} (see problems.py)",
                   "elements": nt, "k": cond["k"],
                   "parallelism": "replicas" if world > 1 else "single-gpu",
                   "l2": "flushed before every timed step (256 MiB write, then a 256 MiB read of another buffer so no dirty lines remain)"},
        "breakdown_ms": cond["breakdown_ms"],
        "apply_dof_per_s": head["apply"]["dof_per_s"], "apply_ms": head["apply"]["ms"],
        "apply_roofline": head["apply"]["roofline"],
        "apply_parity_rel_l2": head["apply"].get("parity_rel_l2_vs_reference"),
        "smoother_roofline": head["jacobi"],
        "pcg": head["pcg"],
        "roofline": cond["roofline"],
        "e2e": {"value": world * nt / (e2e_ms * 1e-3), "unit": "elements/s",
                "h2d_bytes_per_step": W_h.nbytes, "d2h_bytes_per_step": out_bytes,
                "ms_per_step": e2e_ms, "chunks": nch,
                "pcg_solve_e2e_ms": float(np.mean(pcg_e2e)),
                "pcg_solve_e2e_note": "additive PCG to 1e-8 via krylov.cg: rhs H2D from "
                                      "pinned host memory, x D2H, inside the timed region"},
        "gpu_launches": cond["gpu_launches"],
        "clocks": clk,
    }
    if big:
        out["cfg3"] = big
    if micro:
        out["microbench"] = micro
    if stokes:
        out["stokes_gmres"] = stokes
    if cpu_extra:
        out["cpu_solver_baselines"] = cpu_extra
    return out


def cpu_solver_baselines(head):
    """The reference's CPU solver path (oracle port of `driver.py:133-146`:
    scipy CSR `S_free @ v`, ExtendedAsp + AspPreconditioner with cho_solve /
    SuperLU, `krylov.cg`) on the SAME matrices (the GPU's S_T), 1 thread.
    PCG time = reference iterations x (S apply + preconditioner apply),
    extrapolated from the per-application timings (the full solve takes
    ~75 s at cfg2)."""
    import threadpoolctl
    from oracle import mcs_oracle as O
    from paper_2207_08481_b200 import engine
    sys_ = head["_sys"]
    fes, prob = sys_.fes, head["prob"]
    with threadpoolctl.threadpool_limits(1):
        t0 = time.perf_counter()
        ST = engine.unpack_sym(sys_.S_dev.cpu().numpy(), sys_.z["nloc"])
        osys = O.OracleSystem(fes, prob.nu, ST)
        S_free = osys.S_free()
        t_setup = time.perf_counter() - t0
        v = np.random.default_rng(11).standard_normal(S_free.shape[0])
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            S_free @ v
            ts.append(time.perf_counter() - t0)
        t_S = float(np.median(ts))
        out = {"cores": 1, "kind": "port", "S_apply_ms": 1e3 * t_S,
               "S_apply_dof_per_s": S_free.shape[0] / t_S,
               "oracle_setup_s": round(t_setup, 2)}
        for comp in ("additive", "multiplicative"):
            t0 = time.perf_counter()
            M, _ = O.build_preconditioner(fes, osys, prob.nu, comp)
            t_set = time.perf_counter() - t0
            t0 = time.perf_counter()
            M.apply(v)
            t_M = time.perf_counter() - t0
            its = head["pcg"][comp]["reference_iterations"] or head["pcg"][comp]["iterations"]
            out[comp] = {"precond_setup_s": round(t_set, 2), "precond_apply_ms": 1e3 * t_M,
                         "pcg_s_extrapolated": its * (t_S + t_M),
                         "pcg_iterations_used": its,
                         "gpu_speedup_pcg": its * (t_S + t_M) / (head["pcg"][comp]["solve_ms"] * 1e-3)}
    return out


def run_stokes(fes, sys_, prob, dev):
    """Stokes (saddle) mode on the same condensed system: right-preconditioned
    GMRES to rtol 1e-8 with the block triangular saddle preconditioner
    (additive ASP, facet Jacobi), device time by CUDA events."""
    import torch
    from paper_2207_08481_b200 import preconditioners as pc
    from paper_2207_08481_b200.driver import SolverOptions, condensed_rhs, velocity_preconditioner
    from paper_2207_08481_b200.krylov import gmres
    from paper_2207_08481_b200.operators import SaddleOperator
    K = SaddleOperator(sys_)
    vel = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition="additive"))
    P = pc.SaddlePreconditioner(vel, pc.PressureMassPrecond.build(fes, prob.nu), K.B)
    rhs = torch.from_numpy(np.concatenate(condensed_rhs(fes, sys_))).to(dev)
    gmres(K, rhs, P, rtol=1e-8, maxit=1000)          # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    x, rep = gmres(K, rhs, P, rtol=1e-8, maxit=1000)
    e1.record()
    torch.cuda.synchronize()
    return {"composition": "additive", "smoother": "jacobi", "n": K.n,
            "iterations": rep.iterations, "converged": rep.converged,
            "final_res": rep.residuals[-1], "solve_ms": e0.elapsed_time(e1),
            "wall_ms": 1e3 * (time.perf_counter() - t0)}


def run_microbench(args, dev):
    """BASELINE config 5: S = B^T A^-1 B for 1,048,576 independent SPD
    problems (n_s = 60, n_c = 36).  The first 65,536-element chunk is the
    SURVEY §8d NumPy stream itself (default_rng(3): G then B per chunk), the
    other chunks come from the device generator with the same distribution
    (seeded); A = G G^T + 60 I is formed on the device, untimed, and its
    packed lower triangle is the timed input.  Parity: the first 256
    elements against `tests/golden/micro_stream.npz` (the reference idiom
    cho_factor / cho_solve / B^T X, condensation.py:216-224, run on the
    reference's own stack) and 64 random elements of the NumPy chunk
    against the oracle."""
    import torch
    from paper_2207_08481_b200 import engine
    n, m = 60, 36
    count = args.micro_count
    chunk = 65536
    Ap = torch.empty((count, n * (n + 1) // 2), dtype=torch.float64, device=dev)
    B = torch.empty((count, n, m), dtype=torch.float64, device=dev)
    r, c = torch.tril_indices(n, n, device=dev)
    eye = n * torch.eye(n, dtype=torch.float64, device=dev)
    rng = np.random.default_rng(3)
    c0 = min(chunk, count)
    G = torch.from_numpy(rng.standard_normal((c0, n, n))).to(dev)
    B[:c0] = torch.from_numpy(rng.standard_normal((c0, n, m))).to(dev)
    Ap[:c0] = (torch.bmm(G, G.transpose(1, 2)) + eye)[:, r, c]
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    for s in range(c0, count, chunk):
        e = min(count, s + chunk)
        G = torch.randn((e - s, n, n), dtype=torch.float64, device=dev, generator=g)
        B[s:e] = torch.randn((e - s, n, m), dtype=torch.float64, device=dev, generator=g)
        Ap[s:e] = (torch.bmm(G, G.transpose(1, 2)) + eye)[:, r, c]
    del G
    S = torch.empty((count, m * (m + 1) // 2), dtype=torch.float64, device=dev)
    info = torch.empty(count, dtype=torch.int32, device=dev)
    for _ in range(3):
        engine.spd_schur(n, m, Ap, B, out=S, info=info)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        engine.spd_schur(n, m, Ap, B, out=S, info=info)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = float(np.mean(ts))
    flops = n ** 3 / 3 + n * n * m + m * m * n
    out = {"elements": count, "ms": t, "elements_per_s": count / (t * 1e-3),
           "tflops": flops * count / (t * 1e-3) / 1e12,
           "flops_per_element": flops, "failed": int((info != 0).sum().item()),
           "inputs": "first 65,536 elements: SURVEY §8d NumPy stream (default_rng(3)); "
                     "rest: torch Philox, same distribution"}
    peaks = load_peaks()
    out["frac_fp64_peak"] = out["tflops"] / peaks["fp64_tflops"]
    bytes_el = 8 * (n * (n + 1) // 2 + n * m + m * (m + 1) // 2)
    out["hbm_gbs"] = bytes_el * count / (t * 1e-3) / 1e9
    gold = _golden("micro_stream")
    S_h = engine.unpack_sym(S[:256].cpu().numpy(), m)
    if gold is not None:
        ng = min(len(gold["S"]), 256)
        out["max_rel_frob_err_vs_reference_fixture"] = max(
            _rel(S_h[i], gold["S"][i]) for i in range(ng))
        out["reference_fixture_elements"] = ng
    from oracle import mcs_oracle as O
    idx = np.random.default_rng(4).choice(c0, 64, replace=False)
    A_s, B_s = Ap[idx].cpu().numpy(), B[idx].cpu().numpy()
    S_s = engine.unpack_sym(S[idx].cpu().numpy(), m)
    out["max_rel_frob_err_vs_oracle"] = max(
        _rel(S_s[i], O.spd_schur(engine.unpack_sym(A_s[i], n), B_s[i])) for i in range(len(idx)))
    return out


# ----------------------------------------------------------- CPU baselines

_WORKER = {}


def _cpu_init(cfg, n):
    import threadpoolctl
    sys.path.insert(0, ROOT)
    from paper_2207_08481_b200.dofmap import FeSystem
    from paper_2207_08481_b200.problems import baseline_config
    _WORKER["limits"] = threadpoolctl.threadpool_limits(1)
    prob = baseline_config(cfg, n)
    _WORKER["prob"] = prob
    _WORKER["fes"] = FeSystem(prob.mesh, prob.regions, prob.k)


def _cpu_worker(elems):
    """Condense a slice of elements with the oracle (reference algorithm)."""
    from oracle import mcs_oracle as O
    prob, fes = _WORKER["prob"], _WORKER["fes"]
    t0 = time.perf_counter()
    for t in elems:
        blocks = O.element_blocks(fes, t, prob.nu, None)
        S_T, _ = O.condense_element(*blocks[:5])
        O.double_schur_element(S_T, prob.k)
    return time.perf_counter() - t0, len(elems)


class CpuCondenser:
    """The reference algorithm on `procs` host processes; rate = elements /
    wall time of the slowest worker (setup excluded)."""

    def __init__(self, cfg, n, procs):
        from concurrent.futures import ProcessPoolExecutor
        n = n or {1: 16, 2: 128, 3: 256}[cfg]
        self.n, self.procs = n, procs
        self.pool = None
        if procs > 1:
            self.pool = ProcessPoolExecutor(procs, initializer=_cpu_init, initargs=(cfg, n))
        else:
            _cpu_init(cfg, n)
        self.rng = np.random.default_rng(5)

    def rate(self, sample):
        nt = 2 * self.n * self.n
        elems = np.sort(self.rng.choice(nt, size=min(sample, nt), replace=False))
        parts = [elems[i::self.procs] for i in range(self.procs)]
        if self.pool is None:
            dt, cnt = _cpu_worker(parts[0])
            return cnt / dt, cnt
        res = list(self.pool.map(_cpu_worker, parts))
        return len(elems) / max(r[0] for r in res), len(elems)

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (the oracle port of
    assembly.py:49-91 + condensation.py:159-224: quadrature blocks, LU
    condensation, double Schur) on every host core, one step = ALL elements
    of the workload (timed, not extrapolated)."""
    if rank != 0:
        return None
    procs = os.cpu_count() or 1
    cc = CpuCondenser(args.cfg, args.n, procs)
    nt = 2 * cc.n * cc.n
    per_step = min(nt, args.ref_elements or nt)
    for _ in range(args.warmup):
        cc.rate(min(per_step, 8 * procs))
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cc.rate(per_step)
        times.append(time.perf_counter() - t0)
    cc.close()
    ms = 1e3 * float(np.mean(times))
    value = per_step / (ms * 1e-3)
    sample = (f"{per_step} of {nt} cfg{args.cfg} elements per step (quadrature blocks + LU "
              f"condensation + double Schur, oracle/mcs_oracle.py), {procs} processes")
    return {"metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded SURVEY §8d generators)",
            "config": {"workload": WORKLOAD if args.cfg == 2 else f"cfg{args.cfg} (see problems.py)",
                       "elements": nt, "k": {1: 2, 2: 4, 3: 6}[args.cfg],
                       "parallelism": f"{procs} host processes"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "elements/s", "cores": procs,
                             "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None, help="grid size (default: the config's)")
    ap.add_argument("--cfg", type=int, default=2, choices=[1, 2, 3],
                    help="BASELINE config of the bench workload (default 2 = configs[1])")
    ap.add_argument("--no-micro", dest="micro", action="store_false")
    ap.add_argument("--e2e-chunks", type=int, default=4,
                    help="element chunks of the e2e step (D2H of chunk c overlaps chunk c+1)")
    ap.add_argument("--no-stokes", dest="stokes", action="store_false",
                    help="skip the Stokes-mode GMRES solve")
    ap.add_argument("--no-cfg3", dest="cfg3", action="store_false",
                    help="skip the config-3 (k = 6) block")
    ap.add_argument("--no-cpu-solver", dest="cpu_solver", action="store_false",
                    help="skip the CPU S-apply / preconditioner / PCG baselines")
    ap.add_argument("--micro-count", type=int, default=1 << 20)
    ap.add_argument("--cpu-sample", type=int, default=3072)
    ap.add_argument("--ref-elements", type=int, default=0,
                    help="reference arm: elements per step (default: all)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    out = run_ours(args, rank, world)
    if rank == 0:
        # CPU baseline: the reference algorithm (oracle port), 1 core, bounded sample
        cc = CpuCondenser(args.cfg, args.n, 1)
        v, cnt = cc.rate(args.cpu_sample)
        out["cpu_baseline"] = {"value": v, "unit": "elements/s", "cores": 1, "kind": "port",
                               "sample": f"{cnt} random cfg{args.cfg} elements, quadrature blocks + "
                                         "LU condensation + double Schur, 1 thread"}
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
