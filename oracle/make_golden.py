"""Generate tests/golden/*.npz by running the REFERENCE implementation.

TEST INFRASTRUCTURE ONLY.  Run in the build container (where the read-only
reference lives at /root/reference); the GPU box never runs this, it only
reads the committed fixtures:

    python oracle/make_golden.py

Every fixture is produced through the reference's own public API
(`mcstokes.mesh`, `dofmap.FeSystem`, `assembly.assemble_element_blocks`,
`condensation.condense_sigma_omega` / `double_schur`,
`preconditioners.*`, `driver.velocity_preconditioner`, `krylov.cg`), on the
seeded inputs of `paper_2207_08481_b200.problems` (SURVEY §8d protocol).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = os.environ.get("MCS_REFERENCE_SRC", "/root/reference/pkg/src")
OUT = os.path.join(ROOT, "tests", "golden")


def _ref():
    sys.path.insert(0, REF)
    import mcstokes  # noqa: F401
    from mcstokes import assembly, condensation, dofmap, driver, krylov, mesh
    from mcstokes import preconditioners as pc
    return dict(assembly=assembly, condensation=condensation, dofmap=dofmap,
                driver=driver, krylov=krylov, mesh=mesh, pc=pc)


def _csr(prefix, A, out):
    A = A.tocsr()
    A.sort_indices()
    out[prefix + "_data"] = A.data
    out[prefix + "_indices"] = A.indices.astype(np.int32)
    out[prefix + "_indptr"] = A.indptr.astype(np.int64)
    out[prefix + "_shape"] = np.array(A.shape)


def case(R, name, cfg, n, with_matrices=True, comps=("additive", "multiplicative")):
    sys.path.insert(0, ROOT)
    from paper_2207_08481_b200.problems import baseline_config
    prob = baseline_config(cfg, n)
    m = R["mesh"].from_arrays(prob.mesh.vertices, prob.mesh.triangles)
    eps = 1e-12
    key = "tilde_neumann" if cfg == 3 else "neumann"
    regions = R["mesh"].classify_boundary(
        m, dirichlet=lambda x: x[0] < 1 - eps, **{key: lambda x: x[0] >= 1 - eps})
    fes = R["dofmap"].FeSystem(m, regions, prob.k)
    out = dict(k=prob.k, nu=prob.nu, n=n, cfg=cfg)
    out["vertices"], out["triangles"] = m.vertices, m.triangles
    for a in ("facets", "facet_tri", "facet_normal", "facet_tangent",
              "facet_length", "facet_start", "tri_facets"):
        out["mesh_" + a] = getattr(m, a)
    out["bdm_coef"], out["sigma_coef"] = fes.bdm.coef, fes.sigma.coef
    out["v_l2g"], out["v_signs"] = fes.dof_v.loc2glob, fes.dof_v.signs
    out["h_l2g"], out["h_signs"] = fes.dof_vhat.loc2glob, fes.dof_vhat.signs
    out["vv_free"], out["vbar_free"] = fes.vv_free, fes.dof_vbar.is_free

    blocks = R["assembly"].all_element_blocks(fes, prob.nu, prob.body_force)
    if with_matrices:
        for b in ("msig", "bws", "bus", "bhs", "adiv", "bpu", "load"):
            out["eb_" + b] = np.array([getattr(eb, b) for eb in blocks])
    sys_ = R["condensation"].condense_sigma_omega(fes, prob.nu, prob.body_force,
                                                  blocks=blocks)
    R["condensation"].double_schur(sys_)
    if with_matrices:
        _csr("S", sys_.S, out)
        _csr("Sd", sys_.Sd, out)
        out["ext"] = np.array(sys_.ext)
        out["soo"] = np.array(sys_.soo_dense)
        out["recovery"] = np.array(sys_.recovery)
    out["load_vv"] = sys_.load
    pc = R["pc"]
    E = pc.build_embedding(fes)
    Ec = pc.embedding_cpl(fes, sys_, E)
    _csr("Ec", Ec, out)
    coarse = pc.build_coarse(fes, prob.nu, penalty_C=4.0)
    _csr("coarse", coarse.matrix, out)
    blocks_s = pc.facet_blocks_schur(fes, sys_)
    out["fblk_ptr"] = np.cumsum([0] + [len(b) for b in blocks_s])
    out["fblk_idx"] = np.concatenate(blocks_s)

    free = fes.vv_free
    S_free = sys_.S[free][:, free].tocsr()
    rhs_u, _ = R["driver"].condensed_rhs(fes, sys_)
    out["rhs_u"] = rhs_u
    rng = np.random.default_rng(11)
    v = rng.standard_normal(S_free.shape[0])
    out["probe_v"] = v
    out["probe_Sv"] = S_free @ v
    for comp in comps:
        opts = R["driver"].SolverOptions(mode="elliptic", target="Sd",
                                         smoother="jacobi", composition=comp,
                                         rtol=1e-8, maxit=2000)
        M = R["driver"].velocity_preconditioner(fes, sys_, prob.nu, opts)
        out[f"probe_M_{comp}"] = M(v)
        x, rep = R["krylov"].cg(lambda u: S_free @ u, rhs_u, M, rtol=1e-8, maxit=2000)
        out[f"cg_{comp}_iters"] = rep.iterations
        out[f"cg_{comp}_res"] = np.array(rep.residuals)
        out[f"cg_{comp}_x"] = x
        # the multiplicative composition's power-iteration scale
        free_cpl = sys_.free_mask_cpl()
        A = sys_.Sd[free_cpl][:, free_cpl].tocsr()
        sm = pc.FacetBlockSmoother(A, blocks_s, "jacobi")
        asp = pc.AspPreconditioner(A, sm, Ec, coarse, comp, 1)
        out[f"jacobi_scale_{comp}"] = asp.jacobi_scale
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **out)
    print(f"{path}: {os.path.getsize(path) / 1e3:.0f} kB, cg iters",
          {c: int(out[f'cg_{c}_iters']) for c in comps})


def stokes_case(R, name, cfg, n, comps=("additive", "multiplicative")):
    """Stokes (saddle) mode through the reference's own pieces, exactly as
    `driver.solve_stokes` wires them (driver.py:148-160): K = [[S, B^T],
    [B, 0]] on free dofs, SaddlePreconditioner(velocity_preconditioner,
    PressureMassPrecond, B_free), krylov.gmres."""
    import scipy.sparse as sp
    sys.path.insert(0, ROOT)
    from paper_2207_08481_b200.problems import baseline_config
    prob = baseline_config(cfg, n)
    m = R["mesh"].from_arrays(prob.mesh.vertices, prob.mesh.triangles)
    eps = 1e-12
    key = "tilde_neumann" if cfg == 3 else "neumann"
    regions = R["mesh"].classify_boundary(
        m, dirichlet=lambda x: x[0] < 1 - eps, **{key: lambda x: x[0] >= 1 - eps})
    fes = R["dofmap"].FeSystem(m, regions, prob.k)
    sys_ = R["condensation"].condense_sigma_omega(fes, prob.nu, prob.body_force)
    R["condensation"].double_schur(sys_)
    free = fes.vv_free
    S_free = sys_.S[free][:, free].tocsr()
    B_free = sys_.B[:, free].tocsr()
    K = sp.bmat([[S_free, B_free.T], [B_free, None]], format="csr")
    rhs_u, rhs_p = R["driver"].condensed_rhs(fes, sys_)
    rhs = np.concatenate([rhs_u, rhs_p])
    mp = R["pc"].PressureMassPrecond.build(fes, prob.nu)
    out = dict(k=prob.k, nu=prob.nu, n=n, cfg=cfg, rhs=rhs)
    _csr("B", sys_.B, out)
    rng = np.random.default_rng(21)
    v = rng.standard_normal(K.shape[0])
    out["probe_v"], out["probe_Kv"] = v, K @ v
    for comp in comps:
        opts = R["driver"].SolverOptions(mode="stokes", target="Sd", smoother="jacobi",
                                         composition=comp, rtol=1e-8, maxit=500)
        vel = R["driver"].velocity_preconditioner(fes, sys_, prob.nu, opts)
        saddle = R["pc"].SaddlePreconditioner(vel, mp, B_free)
        out[f"probe_P_{comp}"] = saddle.apply(v)
        x, rep = R["krylov"].gmres(lambda u: K @ u, rhs, saddle.apply, rtol=1e-8, maxit=500)
        out[f"gmres_{comp}_iters"] = rep.iterations
        out[f"gmres_{comp}_res"] = np.array(rep.residuals)
        out[f"gmres_{comp}_x"] = x
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **out)
    print(f"{path}: {os.path.getsize(path) / 1e3:.0f} kB, gmres iters",
          {c: int(out[f'gmres_{c}_iters']) for c in comps})


def postcheck_case(R, name, cfg, n):
    """Reference driver.post_checks (driver.py:183-218) on seeded random
    velocity / stress vectors and a fixed residual history."""
    sys.path.insert(0, ROOT)
    from paper_2207_08481_b200.problems import baseline_config
    prob = baseline_config(cfg, n)
    m = R["mesh"].from_arrays(prob.mesh.vertices, prob.mesh.triangles)
    eps = 1e-12
    key = "tilde_neumann" if cfg == 3 else "neumann"
    regions = R["mesh"].classify_boundary(
        m, dirichlet=lambda x: x[0] < 1 - eps, **{key: lambda x: x[0] >= 1 - eps})
    fes = R["dofmap"].FeSystem(m, regions, prob.k)
    rng = np.random.default_rng(31)
    u = rng.standard_normal(fes.dof_v.ndof)
    sigma = rng.standard_normal(fes.dof_sigma.ndof)
    rep = R["krylov"].KrylovReport(residuals=[1.0, 0.5, 0.25, 0.3])
    chk = R["driver"].post_checks(fes, None, u, sigma, rep)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, u=u, sigma=sigma, residuals=np.array(rep.residuals),
                        max_div_scaled=chk["max_div_scaled"], nt_jump_scaled=chk["nt_jump_scaled"],
                        residual_monotone=chk["residual_monotone"])
    print(path, chk)


def microbench(R):
    import scipy.linalg as sla
    sys.path.insert(0, ROOT)
    from paper_2207_08481_b200.problems import microbench_host
    A, B = microbench_host(16, seed=3)
    # the reference idiom of condensation.py:216-224
    S = np.array([B[i].T @ sla.cho_solve(sla.cho_factor(A[i], check_finite=False),
                                         B[i], check_finite=False)
                  for i in range(len(A))])
    path = os.path.join(OUT, "micro.npz")
    np.savez_compressed(path, A=A, B=B, S=S)
    print(path)


def microbench_stream(R, keep=256, chunk=65536):
    """The first `keep` elements of the SURVEY §8d config-5 stream as the
    full-size run draws it: default_rng(3), G for a whole 65,536-element
    chunk, then B for that chunk; S by the reference idiom
    (condensation.py:216-224).  A and B are regenerated by the readers."""
    import scipy.linalg as sla
    rng = np.random.default_rng(3)
    G = rng.standard_normal((chunk, 60, 60))[:keep]
    B = rng.standard_normal((chunk, 60, 36))[:keep]
    A = G @ np.swapaxes(G, 1, 2) + 60 * np.eye(60)
    S = np.array([B[i].T @ sla.cho_solve(sla.cho_factor(A[i], check_finite=False),
                                         B[i], check_finite=False) for i in range(keep)])
    path = os.path.join(OUT, "micro_stream.npz")
    np.savez_compressed(path, S=S, keep=keep, chunk=chunk, seed=3)
    print(path)


def main():
    os.makedirs(OUT, exist_ok=True)
    R = _ref()
    if "--postcheck" in sys.argv:
        postcheck_case(R, "postcheck_c2_n3", 2, 3)
        postcheck_case(R, "postcheck_c3_n2", 3, 2)
        return
    if "--micro-stream" in sys.argv:
        microbench_stream(R)
        return
    if "--stokes" in sys.argv:
        stokes_case(R, "stokes_c1_n2", 1, 2)
        stokes_case(R, "stokes_c2_n3", 2, 3)
        stokes_case(R, "stokes_c3_n2", 3, 2)
        return
    case(R, "c1_n2", 1, 2)
    case(R, "c2_n3", 2, 3)
    case(R, "c3_n2", 3, 2)
    case(R, "cfg1", 1, 16, with_matrices=False)
    microbench(R)
    microbench_stream(R)
    stokes_case(R, "stokes_c1_n2", 1, 2)
    stokes_case(R, "stokes_c2_n3", 2, 3)
    stokes_case(R, "stokes_c3_n2", 3, 2)
    postcheck_case(R, "postcheck_c2_n3", 2, 3)
    postcheck_case(R, "postcheck_c3_n2", 3, 2)


if __name__ == "__main__":
    main()
