"""Full-size (BASELINE config 2 and 3) PCG fixtures from the REFERENCE.

TEST INFRASTRUCTURE ONLY.  Runs in the build container, where the read-only
reference lives at /root/reference; the GPU box only reads the committed
`tests/golden/cfg{2,3}_full.npz`.

    OMP_NUM_THREADS=1 python oracle/make_golden_full.py cfg2   # ~45-60 min
    OMP_NUM_THREADS=1 python oracle/make_golden_full.py cfg3   # memory-lean

Cross-checks of the memory-lean driver against the reference as written
(`MCS_GOLDEN_N` shrinks the grid, `MCS_GOLDEN_OUT` redirects the output):

    python oracle/make_golden_full.py lean2       # lean driver, full cfg2
    MCS_GOLDEN_N=16 python oracle/make_golden_full.py written3 / cfg3

cfg2 runs the reference AS WRITTEN through its own public API
(`FeSystem`, `condense_sigma_omega`, `double_schur`, `condensed_rhs`,
`driver.velocity_preconditioner`, `krylov.cg`, `S_free @ v`), exactly the
wiring of `driver.solve_stokes` elliptic mode (driver.py:133-146).  The one
change is that `preconditioners.build_embedding` (the reference's own
function, ~1000 s at cfg2) is memoised per FeSystem, so the two compositions
do not rebuild the same E.

cfg3 cannot run as written (>70 GB RAM, 5-6 h).  The
memory-lean driver below keeps every reference call that fits and restates
only the three that do not:

* element blocks: the reference's `assemble_element_blocks` (assembly.py:49)
  per element, in 8 forked workers;
* per-element condensation: `condensation.py:161-176` restated line for line
  (same lu_factor / lu_solve / symmetrisation) on each element;
* per-element double Schur: `condensation.py:213-224` on the element-local
  S_T (interior rows are private to one element and carry sign +1, so
  S[gint, gint] = S_T[iint, iint] and S[gint, gl[icpl]]*sg = S_T[iint, icpl]
  exactly);
* S_free @ v: matrix-free sum over elements of P^T D S_T D P v, instead of
  the assembled CSR (7.2e8 COO entries); equal up to summation order;
* S_d assembled from the per-element S_cc - S_oc^T X (COO sum; summation
  order differs from `:225-233` at round-off level);
* E_c: the facet part of `build_embedding` (preconditioners.py:37-63)
  restated; the interior fit (:66-91, the super-linear part) only writes
  interior-bubble rows, which `embedding_cpl` (:101-105) drops.

Everything else is the reference's own code: `FeSystem`, `build_coarse`
(SuperLU), `facet_blocks_schur`, `FacetBlockSmoother`, `AspPreconditioner`
(incl. the power-iteration `jacobi_scale`), `ExtendedAsp`, `embedding_cpl`,
`krylov.cg`.  cfg3 vectors are too large for the repository (57 MB each),
so the fixture keeps full norms plus a seeded sample of 262,144 entries.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = os.environ.get("MCS_REFERENCE_SRC", "/root/reference/pkg/src")
OUT = os.path.join(ROOT, "tests", "golden")
COMPS = ("additive", "multiplicative")
NSAMPLE = 262_144


def _ref():
    sys.path.insert(0, REF)
    sys.path.insert(0, ROOT)
    from mcstokes import (assembly, condensation, dofmap, driver, krylov,  # noqa
                          mesh, preconditioners)
    return dict(assembly=assembly, condensation=condensation, dofmap=dofmap,
                driver=driver, krylov=krylov, mesh=mesh, pc=preconditioners)


def _fes(R, cfg):
    from paper_2207_08481_b200.problems import baseline_config
    prob = baseline_config(cfg, int(os.environ.get("MCS_GOLDEN_N", 0)) or None)
    m = R["mesh"].from_arrays(prob.mesh.vertices, prob.mesh.triangles)
    eps = 1e-12
    key = "tilde_neumann" if cfg == 3 else "neumann"
    regions = R["mesh"].classify_boundary(
        m, dirichlet=lambda x: x[0] < 1 - eps, **{key: lambda x: x[0] >= 1 - eps})
    return prob, R["dofmap"].FeSystem(m, regions, prob.k)


def sample_index(n, seed=5):
    """Seeded sample of entries kept from the cfg3 vectors (sorted, unique)."""
    rng = np.random.default_rng(seed)
    return np.unique(rng.integers(0, n, size=NSAMPLE))


def probe_vector(n, seed=11):
    return np.random.default_rng(seed).standard_normal(n)


# ------------------------------------------------------------------ config 2


def as_written(cfg=2):
    R = _ref()
    pc = R["pc"]
    orig = pc.build_embedding
    cache = {}

    def build_embedding_memo(fes):
        if id(fes) not in cache:
            cache[id(fes)] = orig(fes)
        return cache[id(fes)]

    pc.build_embedding = build_embedding_memo
    tm = {}
    t0 = time.perf_counter()
    prob, fes = _fes(R, cfg)
    tm["fes"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    blocks = R["assembly"].all_element_blocks(fes, prob.nu, prob.body_force)
    tm["element_blocks"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    sys_ = R["condensation"].condense_sigma_omega(fes, prob.nu, prob.body_force,
                                                  blocks=blocks)
    tm["condense"] = time.perf_counter() - t0
    del blocks
    t0 = time.perf_counter()
    R["condensation"].double_schur(sys_)
    tm["double_schur"] = time.perf_counter() - t0
    print("condensed", tm, flush=True)
    free = fes.vv_free
    S_free = sys_.S[free][:, free].tocsr()
    rhs_u, _ = R["driver"].condensed_rhs(fes, sys_)
    v = probe_vector(S_free.shape[0])
    out = dict(cfg=cfg, n=fes.mesh.num_triangles, k=prob.k, nu=prob.nu, rhs_u=rhs_u,
               probe_seed=11)
    out["probe_Sv"] = S_free @ v
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        S_free @ v
        ts.append(time.perf_counter() - t0)
    tm["S_apply_median"] = float(np.median(ts))
    for comp in COMPS:
        opts = R["driver"].SolverOptions(mode="elliptic", target="Sd",
                                         smoother="jacobi", composition=comp,
                                         rtol=1e-8, maxit=2000)
        t0 = time.perf_counter()
        M = R["driver"].velocity_preconditioner(fes, sys_, prob.nu, opts)
        tm[f"precond_setup_{comp}"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        out[f"probe_M_{comp}"] = M(v)
        tm[f"precond_apply_{comp}"] = time.perf_counter() - t0
        out[f"jacobi_scale_{comp}"] = M.__self__.inner.jacobi_scale
        t0 = time.perf_counter()
        x, rep = R["krylov"].cg(lambda u: S_free @ u, rhs_u, M, rtol=1e-8, maxit=2000)
        tm[f"cg_{comp}"] = time.perf_counter() - t0
        out[f"cg_{comp}_iters"] = rep.iterations
        out[f"cg_{comp}_res"] = np.array(rep.residuals)
        out[f"cg_{comp}_x"] = x
        out[f"cg_{comp}_converged"] = rep.converged
        print(comp, rep.iterations, tm, flush=True)
    out["timings_json"] = repr(tm)
    path = os.environ.get("MCS_GOLDEN_OUT") or os.path.join(OUT, "cfg2_full.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path) / 1e6, "MB", tm, flush=True)


def stokes_written(cfg=2, comps=("additive",)):
    """Stokes (saddle) mode at the BASELINE size through the reference as
    written (driver.py:147-161: K = [[S, B^T], [B, 0]] on free dofs,
    SaddlePreconditioner(velocity_preconditioner, PressureMassPrecond),
    krylov.gmres), smoother "jacobi", rtol 1e-8.  Vectors: norms + a seeded
    sample (the full K has 1.26 M unknowns at cfg2)."""
    import scipy.sparse as sp
    R = _ref()
    pc = R["pc"]
    orig = pc.build_embedding
    cache = {}

    def build_embedding_memo(fes):
        if id(fes) not in cache:
            cache[id(fes)] = orig(fes)
        return cache[id(fes)]

    pc.build_embedding = build_embedding_memo
    tm = {}
    prob, fes = _fes(R, cfg)
    t0 = time.perf_counter()
    sys_ = R["condensation"].condense_sigma_omega(fes, prob.nu, prob.body_force)
    R["condensation"].double_schur(sys_)
    tm["condense"] = time.perf_counter() - t0
    free = fes.vv_free
    S_free = sys_.S[free][:, free].tocsr()
    B_free = sys_.B[:, free].tocsr()
    K = sp.bmat([[S_free, B_free.T], [B_free, None]], format="csr")
    rhs_u, rhs_p = R["driver"].condensed_rhs(fes, sys_)
    rhs = np.concatenate([rhs_u, rhs_p])
    mp = pc.PressureMassPrecond.build(fes, prob.nu)
    idx = sample_index(K.shape[0])
    out = dict(cfg=cfg, n=fes.mesh.num_triangles, k=prob.k, nu=prob.nu, sample_idx=idx,
               rhs_norm=np.linalg.norm(rhs), rhs_sample=rhs[idx])
    v = probe_vector(K.shape[0], seed=21)
    Kv = K @ v
    out["probe_Kv_norm"], out["probe_Kv_sample"] = np.linalg.norm(Kv), Kv[idx]
    for comp in comps:
        opts = R["driver"].SolverOptions(mode="stokes", target="Sd", smoother="jacobi",
                                         composition=comp, rtol=1e-8, maxit=1000)
        t0 = time.perf_counter()
        vel = R["driver"].velocity_preconditioner(fes, sys_, prob.nu, opts)
        saddle = pc.SaddlePreconditioner(vel, mp, B_free)
        tm[f"setup_{comp}"] = time.perf_counter() - t0
        Pv = saddle.apply(v)
        out[f"probe_P_{comp}_norm"], out[f"probe_P_{comp}_sample"] = np.linalg.norm(Pv), Pv[idx]
        t0 = time.perf_counter()
        x, rep = R["krylov"].gmres(lambda u: K @ u, rhs, saddle.apply, rtol=1e-8, maxit=1000)
        tm[f"gmres_{comp}"] = time.perf_counter() - t0
        out[f"gmres_{comp}_iters"] = rep.iterations
        out[f"gmres_{comp}_res"] = np.array(rep.residuals)
        out[f"gmres_{comp}_converged"] = rep.converged
        out[f"gmres_{comp}_x_norm"] = np.linalg.norm(x)
        out[f"gmres_{comp}_x_sample"] = x[idx]
        print(comp, rep.iterations, tm, flush=True)
    out["timings_json"] = repr(tm)
    tag = "" if comps == ("additive",) else "_" + "_".join(comps)
    path = os.environ.get("MCS_GOLDEN_OUT") or os.path.join(OUT, f"stokes_cfg{cfg}{tag}_full.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path) / 1e6, "MB", tm, flush=True)


# ------------------------------------------------------------------ config 3

_G = {}


def _cfg3_worker(args):
    """Per-element reference code for elements [lo, hi): blocks
    (assembly.py:49), condensation (condensation.py:161-176), double Schur
    (condensation.py:213-224).  Writes into shared memmaps."""
    import scipy.linalg as sla
    lo, hi = args
    R, fes, prob, mm = _G["R"], _G["fes"], _G["prob"], _G["mm"]
    ns, nw = fes.sigma.ndof, fes.skew.ndof
    nloc_u, nloc_h = fes.bdm.ndof, 3 * fes.k
    nloc = nloc_u + nloc_h
    k = fes.k
    n_em = 3 * (k + 1)
    icpl = np.concatenate([np.arange(n_em), np.arange(nloc_u, nloc_u + nloc_h)])
    iint = np.arange(n_em, nloc_u)
    ST, LD, XX, CH, SD = (np.load(mm[a], mmap_mode="r+") for a in
                          ("ST", "LOAD", "X", "CH", "SD"))
    for t in range(lo, hi):
        eb = R["assembly"].assemble_element_blocks(fes, t, prob.nu, prob.body_force)
        M = np.zeros((ns + nw, ns + nw))
        M[:ns, :ns] = -eb.msig
        M[:ns, ns:] = eb.bws.T
        M[ns:, :ns] = eb.bws
        Bsig = np.zeros((nloc, ns + nw))
        Bsig[:nloc_u, :ns] = eb.bus
        Bsig[nloc_u:, :ns] = eb.bhs
        lu = sla.lu_factor(M, check_finite=False)
        Rm = sla.lu_solve(lu, Bsig.T, check_finite=False)
        S_T = -Bsig @ Rm
        S_T[:nloc_u, :nloc_u] += eb.adiv
        S_T = 0.5 * (S_T + S_T.T)
        ST[t] = S_T
        LD[t] = eb.load
        Soo = S_T[np.ix_(iint, iint)]
        Soc = S_T[np.ix_(iint, icpl)]
        ch = sla.cho_factor(Soo, check_finite=False)
        X = sla.cho_solve(ch, Soc, check_finite=False)
        XX[t] = X
        CH[t] = ch[0]
        assert not ch[1]
        SD[t] = S_T[np.ix_(icpl, icpl)] - Soc.T @ X
    for a in (ST, LD, XX, CH, SD):
        a.flush()
    return hi - lo


def _facet_embedding(fes, k):
    """Facet rows of `build_embedding` (preconditioners.py:37-63) restated."""
    import scipy.sparse as sp
    from mcstokes.basis import shifted_legendre
    mesh = fes.mesh
    qe = fes.quad_edge
    legk = shifted_legendre(k, qe.points)
    rows, cols, vals = [], [], []
    hat = np.vstack([1.0 - qe.points, qe.points])
    tn = set(int(f) for f in fes.regions.tilde_neumann_facets)
    for f in range(mesh.num_facets):
        a = mesh.facet_start[f]
        b = mesh.facets[f, 0] if mesh.facets[f, 0] != a else mesh.facets[f, 1]
        nF, tF = mesh.facet_normal[f], mesh.facet_tangent[f]
        ln = mesh.facet_length[f]
        zero_that = f in tn
        for iv, v in enumerate((a, b)):
            for q in range(k + 1):
                mom = ln * np.sum(qe.weights * hat[iv] * legk[q])
                if abs(mom) < 1e-15:
                    continue
                for c in range(2):
                    rows.append(f * (k + 1) + q)
                    cols.append(2 * v + c)
                    vals.append(mom * nF[c])
            if not zero_that:
                for q in range(k):
                    mom = np.sum(qe.weights * hat[iv] * legk[q])
                    if abs(mom) < 1e-15:
                        continue
                    for c in range(2):
                        rows.append(fes.n_v + f * k + q)
                        cols.append(2 * v + c)
                        vals.append(mom * tF[c])
    return sp.coo_matrix((vals, (rows, cols)),
                         shape=(fes.n_vv, fes.dof_vbar.ndof)).tocsr()


def lean(cfg=3, nproc=8, workdir=None):
    workdir = workdir or f"/tmp/mcs_lean{cfg}"
    import multiprocessing as mp
    import scipy.linalg as sla
    import scipy.sparse as sp
    R = _ref()
    tm = {}
    t0 = time.perf_counter()
    prob, fes = _fes(R, cfg)
    tm["fes"] = time.perf_counter() - t0
    nt = fes.mesh.num_triangles
    k = fes.k
    nloc_u, nloc_h = fes.bdm.ndof, 3 * k
    nloc = nloc_u + nloc_h
    n_em = 3 * (k + 1)
    n_int = nloc_u - n_em
    ncpl = nloc - n_int
    icpl = np.concatenate([np.arange(n_em), np.arange(nloc_u, nloc_u + nloc_h)])
    iint = np.arange(n_em, nloc_u)
    os.makedirs(workdir, exist_ok=True)
    shapes = dict(ST=(nt, nloc, nloc), LOAD=(nt, nloc_u), X=(nt, n_int, ncpl),
                  CH=(nt, n_int, n_int), SD=(nt, ncpl, ncpl))
    mm = {}
    for a, shp in shapes.items():
        mm[a] = os.path.join(workdir, a + ".npy")
        if not os.path.exists(mm[a]) or "--reuse" not in sys.argv:
            np.lib.format.open_memmap(mm[a], mode="w+", dtype=np.float64, shape=shp)
    _G.update(R=R, fes=fes, prob=prob, mm=mm)
    if "--reuse" not in sys.argv:
        t0 = time.perf_counter()
        chunks = [(lo, min(lo + 1024, nt)) for lo in range(0, nt, 1024)]
        with mp.get_context("fork").Pool(nproc) as pool:
            done = 0
            for c in pool.imap_unordered(_cfg3_worker, chunks):
                done += c
                if done % 16384 < 1024:
                    print(f"  elements {done}/{nt} {time.perf_counter() - t0:.0f}s",
                          flush=True)
        tm["elements_parallel"] = time.perf_counter() - t0
    ST, LD, XX, CH, SD = (np.load(mm[a], mmap_mode="r") for a in
                          ("ST", "LOAD", "X", "CH", "SD"))
    ST = np.ascontiguousarray(ST)

    # CondensedSystem fields (condensation.py:147-153, :198-202)
    vv_l2g = np.empty((nt, nloc), dtype=np.int64)
    vv_signs = np.empty((nt, nloc))
    vv_l2g[:, :nloc_u] = fes.dof_v.loc2glob
    vv_l2g[:, nloc_u:] = fes.n_v + fes.dof_vhat.loc2glob
    vv_signs[:, :nloc_u] = fes.dof_v.signs
    vv_signs[:, nloc_u:] = fes.dof_vhat.signs
    load = np.zeros(fes.n_vv)
    np.add.at(load, vv_l2g[:, :nloc_u].ravel(), (LD * vv_signs[:, :nloc_u]).ravel())
    mask_cpl = ~fes.vv_interior
    vv_of_cpl = np.nonzero(mask_cpl)[0]
    cpl_of_vv = -np.ones(fes.n_vv, dtype=np.int64)
    cpl_of_vv[mask_cpl] = np.arange(mask_cpl.sum())
    t0 = time.perf_counter()
    rows = cpl_of_vv[vv_l2g[:, icpl]]
    sgc = vv_signs[:, icpl]
    ii = np.repeat(rows, ncpl, axis=1).ravel()
    jj = np.tile(rows, (1, ncpl)).ravel()
    vv = (np.asarray(SD) * sgc[:, :, None] * sgc[:, None, :]).ravel()
    Sd = sp.coo_matrix((vv, (ii, jj)), shape=(len(vv_of_cpl),) * 2).tocsr()
    del ii, jj, vv
    tm["Sd_assembly"] = time.perf_counter() - t0
    CS = R["condensation"].CondensedSystem
    ext = [np.asarray(XX[t]) for t in range(nt)]
    chols = [(np.asarray(CH[t]), False) for t in range(nt)]
    sys_ = CS(fes=fes, nu=prob.nu, S=None, B=None, load=load, recovery=None,
              vv_l2g=vv_l2g, vv_signs=vv_signs, n_cpl_loc=ncpl, nloc_u=nloc_u,
              Sd=Sd, ext=ext, soo_chol=chols, soo_dense=None,
              cpl_of_vv=cpl_of_vv, vv_of_cpl=vv_of_cpl)
    free = fes.vv_free
    fidx = -np.ones(fes.n_vv, dtype=np.int64)
    fidx[free] = np.arange(free.sum())
    lg_free = fidx[vv_l2g]                            # -1 on constrained dofs
    sg_free = np.where(lg_free >= 0, vv_signs, 0.0)
    lg_safe = np.where(lg_free >= 0, lg_free, 0)
    nfree = int(free.sum())

    def S_free_apply(v):
        """Sum_T P^T D S_T D P v on free dofs (== S[free][:, free] @ v)."""
        xl = v[lg_safe] * sg_free
        yl = np.einsum("tij,tj->ti", ST, xl, optimize=False) * sg_free
        return np.bincount(lg_safe.ravel(), weights=yl.ravel(), minlength=nfree)

    rhs_u = load[free]            # homogeneous Dirichlet: condensed_rhs lift = 0
    pc = R["pc"]
    t0 = time.perf_counter()
    E = _facet_embedding(fes, k)
    Ec = pc.embedding_cpl(fes, sys_, E)
    tm["embedding"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    coarse = pc.build_coarse(fes, prob.nu, penalty_C=4.0)
    tm["coarse"] = time.perf_counter() - t0
    free_cpl = sys_.free_mask_cpl()
    A = Sd[free_cpl][:, free_cpl].tocsr()
    t0 = time.perf_counter()
    blocks = pc.facet_blocks_schur(fes, sys_)
    sm = pc.FacetBlockSmoother(A, blocks, "jacobi")
    tm["smoother"] = time.perf_counter() - t0
    print("setup", tm, flush=True)
    v = probe_vector(nfree)
    idx = sample_index(nfree)
    Sv = S_free_apply(v)
    out = dict(cfg=cfg, n=nt, k=k, nu=prob.nu, sample_idx=idx, probe_seed=11,
               rhs_u_norm=np.linalg.norm(rhs_u), rhs_u_sample=rhs_u[idx],
               probe_Sv_norm=np.linalg.norm(Sv), probe_Sv_sample=Sv[idx])
    t0 = time.perf_counter()
    S_free_apply(v)
    tm["S_apply"] = time.perf_counter() - t0
    for comp in COMPS:
        t0 = time.perf_counter()
        asp = pc.AspPreconditioner(A, sm, Ec, coarse, comp, 1)
        M = pc.ExtendedAsp(sys_, asp).apply
        tm[f"asp_setup_{comp}"] = time.perf_counter() - t0
        out[f"jacobi_scale_{comp}"] = asp.jacobi_scale
        t0 = time.perf_counter()
        Mv = M(v)
        tm[f"precond_apply_{comp}"] = time.perf_counter() - t0
        out[f"probe_M_{comp}_norm"] = np.linalg.norm(Mv)
        out[f"probe_M_{comp}_sample"] = Mv[idx]
        t0 = time.perf_counter()
        x, rep = R["krylov"].cg(S_free_apply, rhs_u, M, rtol=1e-8, maxit=2000)
        tm[f"cg_{comp}"] = time.perf_counter() - t0
        out[f"cg_{comp}_iters"] = rep.iterations
        out[f"cg_{comp}_res"] = np.array(rep.residuals)
        out[f"cg_{comp}_converged"] = rep.converged
        out[f"cg_{comp}_x_norm"] = np.linalg.norm(x)
        out[f"cg_{comp}_x_sample"] = x[idx]
        print(comp, rep.iterations, tm, flush=True)
    out["timings_json"] = repr(tm)
    path = os.environ.get("MCS_GOLDEN_OUT") or os.path.join(OUT, "cfg3_full.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path) / 1e6, "MB", tm, flush=True)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    if "cfg2" in sys.argv:
        as_written(2)
    if "cfg3" in sys.argv:
        lean(3)
    if "lean2" in sys.argv:          # cross-check of the lean driver at cfg2
        lean(2)
    if "written3" in sys.argv:       # cross-check at small cfg3 meshes
        as_written(3)
    if "stokes2" in sys.argv:        # Stokes mode (GMRES) at the full cfg2
        stokes_written(2)
    if "stokes2m" in sys.argv:       # the same, multiplicative composition
        stokes_written(2, comps=("multiplicative",))
