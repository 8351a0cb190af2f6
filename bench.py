#!/usr/bin/env python
"""Benchmark of the B200 condensation + PCG hot path (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): N=128 grid, 32,768
jittered triangles, k=4, nu=1e-2, Fourier body force seed 0.  One *step* is
one condensation pass over all elements on the GPU: element blocks from the
geometry (A1) -> sigma/omega elimination (A3) -> double Schur (A4).
`value` = elements condensed per second, inputs resident in HBM, L2 flushed
before every timed step, device time by CUDA events.  The same run also
measures the condensed-operator apply (DOF/s, A6), the full PCG solve to
rtol 1e-8 (both compositions) and the config-5 SPD-Schur microbench, and
reports the CPU oracle on a bounded sample as `cpu_baseline`.

`--impl reference` times the reference algorithm's CPU restatement
(oracle/mcs_oracle.py: quadrature blocks + LU condensation + double Schur,
condensation.py:159-224 / assembly.py:49-91) on the host cores, process
parallel over elements, on the same workload and metric.

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
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_kernels_*.json")),
                       key=os.path.getmtime, reverse=True):
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


def run_ours(args, rank, world):
    import torch
    from paper_2207_08481_b200 import _abi, engine, refblocks
    from paper_2207_08481_b200.condensation import condense_sigma_omega, double_schur
    from paper_2207_08481_b200.dofmap import FeSystem
    from paper_2207_08481_b200.driver import (SolverOptions, condensed_rhs,
                                               velocity_preconditioner)
    from paper_2207_08481_b200.krylov import cg
    from paper_2207_08481_b200.operators import SOperator
    from paper_2207_08481_b200.problems import baseline_config

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    _abi.lib()
    prob = baseline_config(args.cfg, args.n)
    fes = FeSystem(prob.mesh, prob.regions, prob.k)
    k, nt = prob.k, prob.mesh.num_triangles
    refs = refblocks.build_refs(fes)
    W_h = refblocks.element_weights(fes, prob.nu)
    W = engine.to_dev(W_h)
    prog = [engine.to_dev(a) for a in engine.sblock_program(refs)]
    L = engine.srecord_layout(k)
    unfused_path = args.unfused
    rec = torch.empty((nt, L["len"]), dtype=torch.float64, device=dev) if unfused_path else None
    ST = torch.empty((nt, engine.st_stride(k)), dtype=torch.float64, device=dev)
    ext = torch.empty((nt, _abi.call("mcs_ext_stride", k)), dtype=torch.float64, device=dev)
    Sd = torch.empty((nt, _abi.call("mcs_sd_stride", k)), dtype=torch.float64, device=dev)
    info = torch.empty(nt, dtype=torch.int32, device=dev)
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
    st = _abi.stream(stream)

    fused = k in engine.FUSED_DEGREES and not args.unfused
    gen = k not in engine.FUSED_DEGREES and not args.unfused
    if fused or gen:
        tab = engine.to_dev(engine.fused_tables(refs)[0])

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        if fused:   # A1 + A3 + A4 in one warp-per-element kernel
            _abi.call("mcs_condense_fused", k, nt, _abi.ptr(W), W.shape[1], _abi.ptr(tab),
                      _abi.ptr(ST), _abi.ptr(ext), _abi.ptr(Sd), _abi.ptr(info), st)
            if ev:
                ev[1].record(stream)
                ev[2].record(stream)
                ev[3].record(stream)
            return
        if gen:     # A1 + A3 in one kernel (generation fused), then A4
            if ev:
                ev[1].record(stream)
            _abi.call("mcs_condense_gen", k, nt, _abi.ptr(W), W.shape[1], _abi.ptr(tab),
                      _abi.ptr(ST), _abi.ptr(info), st)
        else:
            engine.element_srecords(nt, W, prog, k, out=rec, stream=stream)
            if ev:
                ev[1].record(stream)
            _abi.call("mcs_condense_struct", k, nt, _abi.ptr(rec), _abi.ptr(ST), _abi.ptr(info), st)
        if ev:
            ev[2].record(stream)
        _abi.call("mcs_double_schur", k, nt, _abi.ptr(ST), _abi.ptr(ext), _abi.ptr(Sd),
                  _abi.ptr(info), st)
        if ev:
            ev[3].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if int(info.abs().sum().item()):
        raise RuntimeError("condensation reported failing elements")
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    clocks = ClockSampler(dev.index)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.2)
    for i in range(args.steps):
        l2_flush(i)                           # L2 flush (256 MiB write + 256 MiB read), untimed
        step(evs[i])
    torch.cuda.synchronize()
    t_a1 = np.array([e[0].elapsed_time(e[1]) for e in evs])
    t_a3 = np.array([e[1].elapsed_time(e[2]) for e in evs])
    t_a4 = np.array([e[2].elapsed_time(e[3]) for e in evs])
    t_step = t_a1 + t_a3 + t_a4
    ms_per_step = max_over_ranks(float(t_step.mean()), world, dev)
    value = world * nt / (ms_per_step * 1e-3)

    # ---- condensed-operator apply (A6) and PCG (A8-A13), same run
    sys_ = double_schur(condense_sigma_omega(fes, prob.nu, prob.body_force))
    S = SOperator(sys_)
    n_free = sys_.maps.n_vv_free
    x = torch.randn(n_free, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    for _ in range(5):
        S.apply(x, out=y)
    napp = max(20, args.steps)
    ev_a = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(napp)]
    for i in range(napp):
        l2_flush(i)
        ev_a[i][0].record(stream)
        S.apply(x, out=y)
        ev_a[i][1].record(stream)
    torch.cuda.synchronize()
    t_apply = float(np.mean([e[0].elapsed_time(e[1]) for e in ev_a]))
    z = refblocks.local_sizes(k)
    apply_bytes = nt * 8 * z["nloc"] * (z["nloc"] + 1) / 2 + 16 * n_free
    peaks_hbm = load_peaks()["hbm_gbs"]
    pcg = {}
    smoother = None
    for comp in ("additive", "multiplicative"):
        t0 = time.perf_counter()
        M = velocity_preconditioner(fes, sys_, prob.nu, SolverOptions(smoother="jacobi", composition=comp))
        torch.cuda.synchronize()
        t_sup = time.perf_counter() - t0
        if smoother is None:
            # facet-block Jacobi apply (A9) alone, L2 flushed, HBM roofline
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
            smoother = {"kernel": f"jacobi_apply_kernel<{bsz}>", "ms": t_jac,
                        "note": "event time incl. launch latency; the kernel alone is ~9 us "
                                "under ncu (profiles/)",
                        "bound": "hbm", "achieved": jac_bytes / (t_jac * 1e-3) / 1e9,
                        "peak": peaks_hbm, "unit": "GB/s",
                        "frac": jac_bytes / (t_jac * 1e-3) / 1e9 / peaks_hbm,
                        "algorithmic_bytes": jac_bytes}
        b_h = condensed_rhs(fes, sys_)[0]
        b = torch.from_numpy(b_h).to(dev)
        cg(S, b, M, rtol=1e-8, maxit=2000)      # warm-up (captures the CUDA graphs)
        torch.cuda.synchronize()
        solves = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            xs, rep = cg(S, b, M, rtol=1e-8, maxit=2000)
            e1.record(stream)
            torch.cuda.synchronize()
            solves.append(e0.elapsed_time(e1))
        pcg[comp] = {"iterations": rep.iterations, "final_res": rep.residuals[-1],
                     "solve_ms": float(np.median(solves)),
                     "ms_per_iteration": float(np.median(solves)) / rep.iterations,
                     "precond_setup_s": round(t_sup, 3),
                     "jacobi_scale": M.inner.jacobi_scale,
                     "reference_iterations": ({"additive": 44} if args.cfg == 2 and not args.n else {}).get(comp)}
    stokes = run_stokes(fes, sys_, prob, dev) if args.stokes else None
    clk = clocks.stop()

    # ---- e2e through the C ABI with host buffers: H2D weights, D2H results
    W_pin = torch.from_numpy(W_h).pin_memory()
    out_bytes = (ST.numel() + Sd.numel() + ext.numel()) * 8
    ST_h = torch.empty(ST.shape, dtype=torch.float64).pin_memory()
    Sd_h = torch.empty(Sd.shape, dtype=torch.float64).pin_memory()
    ext_h = torch.empty(ext.shape, dtype=torch.float64).pin_memory()
    e2e_times = []
    # fused path: the elements go through in chunks; chunk c's results leave
    # for the host on a copy stream (its own DMA engine) while chunk c+1 is
    # condensed, so the step costs the PCIe read-back plus one chunk of compute
    nch = args.e2e_chunks if (fused or gen) else 1
    chk = [0, nt // 3, nt // 2, nt - 1]
    ref_rows = [t[chk].cpu() for t in (ST, ext, Sd)]   # from the full-grid launches above
    bounds = [nt * c // nch for c in range(nch + 1)]
    d2h = torch.cuda.Stream()
    done = [torch.cuda.Event() for _ in range(nch)]

    def e2e_step():
        for c in range(nch):
            a, b = bounds[c], bounds[c + 1]
            W[a:b].copy_(W_pin[a:b], non_blocking=True)
            if nch == 1:
                step()
            elif fused:
                _abi.call("mcs_condense_fused", k, b - a, _abi.ptr(W[a:b]), W.shape[1],
                          _abi.ptr(tab), _abi.ptr(ST[a:b]), _abi.ptr(ext[a:b]),
                          _abi.ptr(Sd[a:b]), _abi.ptr(info[a:b]), st)
            else:   # gen: A1 + A3 kernel, then the double Schur, on the chunk
                _abi.call("mcs_condense_gen", k, b - a, _abi.ptr(W[a:b]), W.shape[1],
                          _abi.ptr(tab), _abi.ptr(ST[a:b]), _abi.ptr(info[a:b]), st)
                _abi.call("mcs_double_schur", k, b - a, _abi.ptr(ST[a:b]), _abi.ptr(ext[a:b]),
                          _abi.ptr(Sd[a:b]), _abi.ptr(info[a:b]), st)
            done[c].record(stream)
            d2h.wait_event(done[c])
            with torch.cuda.stream(d2h):
                ST_h[a:b].copy_(ST[a:b], non_blocking=True)
                Sd_h[a:b].copy_(Sd[a:b], non_blocking=True)
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
    # the host copies are the device results (chunked launches included)
    if not all(torch.equal(h[chk], r) for h, r in zip((ST_h, ext_h, Sd_h), ref_rows)):
        raise RuntimeError("e2e host buffers differ from the device results")

    # ---- config-5 microbench (SPD Schur S = B^T A^-1 B, n_s=60, n_c=36)
    micro = run_microbench(args, dev) if args.micro else None

    peaks = load_peaks()
    f_cond, f_ds = flops_per_element(k)
    if fused:
        # the fused kernel is the whole step: A1 + A3 + A4
        f_kern = flops_structured(k)
        t_kern = t_step.mean()
        kname, kpref = f"condense_fused (A1+A3+A4), k={k}", f"condense_fused_kernel<{k},"
    else:
        t_kern = t_a3.mean()
        kname, kpref = ((f"condense_gen (A1+A3), k={k}", f"condense_gen_kernel<{k},") if gen else
                        (f"condense_struct (A3), k={k}", f"condense_struct_kernel<{k},"))
        z_ = refblocks.local_sizes(k)
        ny_ = k * (k + 1) + 3 * k
        f_kern = (z_["nloc"] * (z_["nloc"] + 1) * ny_ + z_["nloc"] * (12 * (k * (k + 1) // 2)
                  + 3 * k * (3 * k + 1)))
    achieved = f_kern * nt / (t_kern * 1e-3) / 1e12
    roofline = {"bound": "tensor", "pipe": "FP64 tensor cores (DMMA m8n8k4) + FP64 FMA",
                "kernel": kname, "achieved": achieved,
                "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                "frac": achieved / peaks["fp64_tflops"] if peaks["fp64_tflops"] else None,
                "flops_per_element": f_kern,
                "dense_equivalent_flops_per_element": f_cond + (f_ds if fused else 0),
                "dense_equivalent_tflops": (f_cond + (f_ds if fused else 0)) * nt
                / (t_kern * 1e-3) / 1e12,
                "traffic": ncu_traffic(kpref),
                "peak_source": "profiles/fp64_peak_r01.json (measured DMMA/DFMA max)"}
    out = {
        "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded SURVEY §8d generators)",
        "config": {"workload": WORKLOAD if args.cfg == 2 else f"cfg{args.cfg} (see problems.py)",
                   "elements": nt, "k": k,
                   "parallelism": "replicas" if world > 1 else "single-gpu",
                   "l2": "flushed before every timed step (256 MiB write, then a 256 MiB read of another buffer so no dirty lines remain)"},
        "breakdown_ms": {"A1_blocks": float(t_a1.mean()), "A3_condense": float(t_a3.mean()),
                         "A4_double_schur": float(t_a4.mean())},
        "apply_dof_per_s": n_free / (t_apply * 1e-3), "apply_ms": t_apply,
        "apply_roofline": {"bound": "hbm", "achieved": apply_bytes / (t_apply * 1e-3) / 1e9,
                           "peak": peaks["hbm_gbs"], "unit": "GB/s",
                           "frac": apply_bytes / (t_apply * 1e-3) / 1e9 / peaks["hbm_gbs"],
                           "traffic": ncu_traffic(f"elem_apply_kernel<{z['nloc']},")},
        "smoother_roofline": smoother,
        "pcg": pcg,
        "roofline": roofline,
        "e2e": {"value": world * nt / (e2e_ms * 1e-3), "unit": "elements/s",
                "h2d_bytes_per_step": W_h.nbytes, "d2h_bytes_per_step": out_bytes,
                "ms_per_step": e2e_ms, "chunks": nch},
        "gpu_launches": (1 if fused else (2 if gen else 3)) * args.steps,
        "clocks": clk,
    }
    if micro:
        out["microbench"] = micro
    if stokes:
        out["stokes_gmres"] = stokes
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
    import torch
    from paper_2207_08481_b200 import engine
    n, m = 60, 36
    count = args.micro_count
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    Ap = torch.empty((count, n * (n + 1) // 2), dtype=torch.float64, device=dev)
    B = torch.empty((count, n, m), dtype=torch.float64, device=dev)
    r, c = torch.tril_indices(n, n, device=dev)
    chunk = 65536
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        G = torch.randn((e - s, n, n), dtype=torch.float64, device=dev, generator=g)
        B[s:e] = torch.randn((e - s, n, m), dtype=torch.float64, device=dev, generator=g)
        A = torch.bmm(G, G.transpose(1, 2)) + n * torch.eye(n, dtype=torch.float64, device=dev)
        Ap[s:e] = A[:, r, c]
        del G, A
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
    # parity on a sample vs the CPU oracle
    from oracle import mcs_oracle as O
    idx = np.random.default_rng(4).choice(count, 64, replace=False)
    A_s = Ap[idx].cpu().numpy()
    B_s = B[idx].cpu().numpy()
    S_s = engine.unpack_sym(S[idx].cpu().numpy(), m)
    worst = 0.0
    for i in range(len(idx)):
        Af = engine.unpack_sym(A_s[i], n)
        ref = O.spd_schur(Af, B_s[i])
        worst = max(worst, np.linalg.norm(S_s[i] - ref) / np.linalg.norm(ref))
    bytes_el = 8 * (n * (n + 1) // 2 + n * m + m * (m + 1) // 2)
    peaks = load_peaks()
    return {"elements": count, "ms": t, "elements_per_s": count / (t * 1e-3),
            "tflops": flops * count / (t * 1e-3) / 1e12,
            "frac_fp64_peak": flops * count / (t * 1e-3) / 1e12 / peaks["fp64_tflops"],
            "hbm_gbs": bytes_el * count / (t * 1e-3) / 1e9,
            "max_rel_frob_err_vs_oracle": worst, "failed": int((info != 0).sum().item())}


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
    """--impl reference: the reference's CPU algorithm (oracle port)."""
    if rank != 0:
        return None
    procs = os.cpu_count() or 1
    cc = CpuCondenser(args.cfg, args.n, procs)
    vals = []
    for _ in range(args.warmup):
        cc.rate(4 * procs)
    for _ in range(args.steps):
        v, cnt = cc.rate(args.ref_sample_per_core * procs)
        vals.append(v)
    cc.close()
    value = float(np.mean(vals))
    sample = (f"{args.ref_sample_per_core * procs} random elements of cfg{args.cfg} per step "
              f"(quadrature blocks + LU condensation + double Schur, oracle/mcs_oracle.py)")
    return {"metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * 2 * cc.n * cc.n / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded SURVEY §8d generators)",
            "config": {"workload": WORKLOAD if args.cfg == 2 else f"cfg{args.cfg} (see problems.py)",
                       "elements": 2 * cc.n * cc.n, "k": {1: 2, 2: 4, 3: 6}[args.cfg],
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
    ap.add_argument("--unfused", action="store_true",
                    help="k <= 4: time the three-kernel path instead of the fused kernel")
    ap.add_argument("--micro-count", type=int, default=1 << 20)
    ap.add_argument("--cpu-sample", type=int, default=3072)
    ap.add_argument("--ref-sample-per-core", type=int, default=32)
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
