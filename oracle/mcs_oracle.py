"""CPU oracle for the condensation + PCG hot path.  TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its CPU-baseline /
`--impl reference` leg) may import this module, and only as the checker or
the timed CPU reference.  The product path (`paper_2207_08481_b200`) never
imports it: with the CUDA library missing the product raises instead of
falling back here.

Each function restates one step of the reference (`mcstokes`, pure
NumPy/SciPy, read-only at /root/reference) line for line in arithmetic, with
the reference call it follows cited as file:line.  The restatement is pinned
(`tests/test_oracle_golden.py`) against golden vectors that
`oracle/make_golden.py` produced by running the reference itself in the
build container; the GPU parity tests then compare the CUDA path with this
oracle on identical seeded inputs.

Inputs are plain arrays plus an object exposing the reference `FeSystem`
attribute names (the product's host `FeSystem` or the reference's own).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class NegativeCurvatureError(Exception):
    pass


# ----------------------------------------------------------- element blocks


def element_blocks(fes, t, nu, body_force=None):
    """Quadrature element blocks; follows `assembly.py:49-91`."""
    w = fes.quad_tri.weights * fes.detJ[t]
    sig = np.einsum("il,splm,jm->spij", fes.JinvT[t], fes.tab_sigma, fes.J[t])
    sdiv = np.einsum("ij,spj->spi", fes.JinvT[t], fes.tab_sigma_div)
    u = np.einsum("ij,upj->upi", fes.J[t], fes.tab_u) / fes.detJ[t]
    udiv = fes.tab_u_div / fes.detJ[t]
    msig = np.einsum("spij,p,zpij->sz", sig, w, sig) / nu
    msig = 0.5 * (msig + msig.T)                                  # :62
    bws = np.einsum("wp,p,sp->ws", fes.tab_w, w,
                    0.5 * (sig[:, :, 1, 0] - sig[:, :, 0, 1]))    # :64-65
    bus = np.einsum("upi,p,spi->us", u, w, sdiv)                  # :66
    adiv = 0.5 * nu * np.einsum("up,p,vp->uv", udiv, w, udiv)     # :67
    adiv = 0.5 * (adiv + adiv.T)
    k = fes.k
    bhs = np.zeros((3 * k, fes.sigma.ndof))
    for le in range(3):                                           # :72-83
        f = fes.edge_facet[t, le]
        sE = np.einsum("il,splm,jm->spij", fes.JinvT[t],
                       fes.tab_sigma_edge[:, le], fes.J[t])
        uE = np.einsum("ij,upj->upi", fes.J[t], fes.tab_u_edge[:, le]) / fes.detJ[t]
        n = fes.edge_normal_out[t, le]
        we = fes.quad_edge.weights * fes.edge_len[t, le]
        snn = np.einsum("i,spij,j->sp", n, sE, n)
        bus -= np.einsum("up,p,sp->us", uE @ n, we, snn)
        tsn = np.einsum("i,spij,j->sp", fes.mesh.facet_tangent[f], sE,
                        fes.mesh.facet_normal[f])
        bhs[le * k:(le + 1) * k] = -fes.edge_sign[t, le] * np.einsum(
            "hp,p,sp->hs", fes.tab_leg_edge[:k], we, tsn)
    load = np.zeros(fes.bdm.ndof)
    if body_force is not None:                                    # :85-89
        X = fes.origin[t] + fes.quad_tri.points @ fes.J[t].T
        F = np.array([body_force(x) for x in X])
        load = np.einsum("upi,p,pi->u", u, w, F)
    return msig, bws, bus, bhs, adiv, load


# ------------------------------------------------------------ condensation


def condense_element(msig, bws, bus, bhs, adiv):
    """S_T and R of one element by LU of the local saddle block; follows
    `condensation.py:161-176` (same lu_factor/lu_solve, same symmetrisation).
    Raises like `:170-172`."""
    ns, nw = msig.shape[0], bws.shape[0]
    nu_l = bus.shape[0]
    nloc = nu_l + bhs.shape[0]
    M = np.zeros((ns + nw, ns + nw))
    M[:ns, :ns] = -msig
    M[:ns, ns:] = bws.T
    M[ns:, :ns] = bws
    Bsig = np.zeros((nloc, ns + nw))
    Bsig[:nu_l, :ns] = bus
    Bsig[nu_l:, :ns] = bhs
    lu = sla.lu_factor(M, check_finite=False)
    if np.any(np.diag(lu[0]) == 0):
        raise RuntimeError("singular local stress block")
    R = sla.lu_solve(lu, Bsig.T, check_finite=False)
    S = -Bsig @ R
    S[:nu_l, :nu_l] += adiv
    return 0.5 * (S + S.T), R


def local_splits(k):
    """(icpl, iint) of the local vv layout; `condensation.py:124-133`."""
    n_em, nu_l, nh = 3 * (k + 1), (k + 1) * (k + 2), 3 * k
    icpl = np.concatenate([np.arange(n_em), np.arange(nu_l, nu_l + nh)])
    return icpl, np.arange(n_em, nu_l)


def double_schur_element(S_T, k):
    """Per-element S_oo, X = S_oo^-1 S_oc and Sd_T = S_cc - S_oc^T X on the
    element-local S_T; follows `condensation.py:212-224` (rows of interior
    dofs are element-private, so S[gint, .] restricted to the element equals
    S_T up to the +-1 signs, which square away)."""
    icpl, iint = local_splits(k)
    Soo = S_T[np.ix_(iint, iint)]
    Soc = S_T[np.ix_(iint, icpl)]
    try:
        ch = sla.cho_factor(Soo, check_finite=False)
    except sla.LinAlgError as exc:
        raise RuntimeError("interior velocity block not SPD") from exc
    X = sla.cho_solve(ch, Soc, check_finite=False)
    Sd = S_T[np.ix_(icpl, icpl)] - Soc.T @ X
    return Soo, X, Sd


def recover_stress(fes, R_list, x_full):
    """Element-wise (sigma, omega) = -R_T u_T; follows `condensation.py:64-74`
    (sigma / omega dofs are element-local, numbered element-major)."""
    l2g, sg = vv_maps(fes)
    ns, nw = R_list[0].shape[0] - fes.k * (fes.k + 1) // 2, fes.k * (fes.k + 1) // 2
    sig = np.empty(len(R_list) * ns)
    wv = np.empty(len(R_list) * nw)
    for t, R in enumerate(R_list):
        so = -R @ (x_full[l2g[t]] * sg[t])
        sig[t * ns:(t + 1) * ns] = so[:ns]
        wv[t * nw:(t + 1) * nw] = so[ns:]
    return sig, wv


def vv_maps(fes):
    """Per-element combined (V, Vhat) local->global map and signs;
    `condensation.py:147-153`."""
    l2g = np.concatenate([fes.dof_v.loc2glob, fes.n_v + fes.dof_vhat.loc2glob], 1)
    sg = np.concatenate([fes.dof_v.signs, fes.dof_vhat.signs], 1)
    return l2g, sg


def assemble(n, l2g, sg, mats):
    """Sum of signed element matrices into CSR; `assembly.py:99-117`."""
    nt, m = l2g.shape
    vals = mats * sg[:, :, None] * sg[:, None, :]
    I = np.repeat(l2g, m, axis=1).ravel()
    J = np.tile(l2g, (1, m)).ravel()
    return sp.coo_matrix((vals.ravel(), (I, J)), shape=(n, n)).tocsr()


def cpl_numbering(fes):
    """vv_of_cpl / cpl_of_vv; `condensation.py:199-202`."""
    mask = ~fes.vv_interior
    vv_of_cpl = np.flatnonzero(mask)
    cpl_of_vv = -np.ones(fes.n_vv, dtype=np.int64)
    cpl_of_vv[mask] = np.arange(mask.sum())
    return vv_of_cpl, cpl_of_vv


class OracleSystem:
    """Everything the elliptic PCG needs, built the reference way."""

    def __init__(self, fes, nu, S_T, load=None):
        k = fes.k
        self.fes, self.nu, self.k = fes, nu, k
        self.S_T = S_T
        self.l2g, self.sg = vv_maps(fes)
        self.S = assemble(fes.n_vv, self.l2g, self.sg, S_T)
        self.load = np.zeros(fes.n_vv)
        if load is not None:                                      # :182
            nu_l = fes.bdm.ndof
            np.add.at(self.load, self.l2g[:, :nu_l].ravel(),
                      (load * self.sg[:, :nu_l]).ravel())
        icpl, iint = local_splits(k)
        self.icpl, self.iint = icpl, iint
        parts = [double_schur_element(S, k) for S in S_T]
        self.Soo = np.array([p[0] for p in parts])
        self.X = np.array([p[1] for p in parts])
        self.Sd_T = np.array([p[2] for p in parts])
        self.chol = [sla.cho_factor(s, check_finite=False) for s in self.Soo]
        self.vv_of_cpl, self.cpl_of_vv = cpl_numbering(fes)
        rows = self.cpl_of_vv[self.l2g[:, icpl]]
        self.Sd = assemble(len(self.vv_of_cpl), rows, self.sg[:, icpl], self.Sd_T)
        self.free_vv = fes.vv_free
        self.free_cpl = fes.vv_free[self.vv_of_cpl]

    def S_free(self):
        f = self.free_vv
        return self.S[f][:, f].tocsr()

    def Sd_free(self):
        f = self.free_cpl
        return self.Sd[f][:, f].tocsr()

    def rhs(self):
        """`driver.py:105-110` (velocity part)."""
        return (self.load - self.S @ self.fes.vv_values)[self.free_vv]


# ---------------------------------------------------------- preconditioner


def facet_blocks_schur(fes, sys_):
    """`preconditioners.py:266-280`."""
    k = fes.k
    idx = -np.ones(len(sys_.free_cpl), dtype=np.int64)
    idx[sys_.free_cpl] = np.arange(sys_.free_cpl.sum())
    out = []
    for f in range(fes.mesh.num_facets):
        dofs = [sys_.cpl_of_vv[f * (k + 1) + q] for q in range(k + 1)]
        dofs += [sys_.cpl_of_vv[fes.n_v + f * k + q] for q in range(k)]
        b = idx[np.array(dofs)]
        b = b[b >= 0]
        if len(b):
            out.append(np.unique(b))
    return out


class Jacobi:
    """Block Jacobi of `preconditioners.py:186-206` (variant "jacobi")."""

    def __init__(self, A, blocks):
        self.blocks = blocks
        self.factors = [sla.cho_factor(A[np.ix_(b, b)].toarray(), check_finite=False)
                        for b in blocks]

    def apply(self, r):
        x = np.zeros_like(r)
        for b, f in zip(self.blocks, self.factors):
            x[b] += sla.cho_solve(f, r[b], check_finite=False)
        return x


def embedding_cpl(fes, sys_):
    """Coupling rows of the P1 -> (V, Vhat) embedding restricted to free
    dofs: the facet loop of `preconditioners.py:40-63` followed by
    `embedding_cpl` (`:101-105`).  The interior-bubble fit (`:66-91`) only
    produces bubble rows, which `embedding_cpl` drops."""
    from scipy.special import eval_legendre  # noqa: F401  (documentation)
    m, k = fes.mesh, fes.k
    s, w = fes.quad_edge.points, fes.quad_edge.weights
    z = 2.0 * s - 1.0
    P = [np.ones_like(z), z]
    for n in range(1, k):
        P.append(((2 * n + 1) * z * P[n] - n * P[n - 1]) / (n + 1))
    leg = np.array(P[:k + 1]) * np.sqrt(2.0 * np.arange(k + 1) + 1.0)[:, None]
    hat = np.vstack([1.0 - s, s])
    rows, cols, vals = [], [], []
    for f in range(m.num_facets):
        a = m.facet_start[f]
        b = m.facets[f, 0] if m.facets[f, 0] != a else m.facets[f, 1]
        nF, tF, ln = m.facet_normal[f], m.facet_tangent[f], m.facet_length[f]
        tilde = f in fes.regions.tilde_neumann_facets
        for iv, v in enumerate((a, b)):
            for q in range(k + 1):
                mom = ln * np.sum(w * hat[iv] * leg[q])
                if abs(mom) >= 1e-15:
                    for c in range(2):
                        rows.append(f * (k + 1) + q); cols.append(2 * v + c)
                        vals.append(mom * nF[c])
            if not tilde:
                for q in range(k):
                    mom = np.sum(w * hat[iv] * leg[q])
                    if abs(mom) >= 1e-15:
                        for c in range(2):
                            rows.append(fes.n_v + f * k + q); cols.append(2 * v + c)
                            vals.append(mom * tF[c])
    E = sp.coo_matrix((vals, (rows, cols)),
                      shape=(fes.n_vv, fes.dof_vbar.ndof)).tocsr()
    return E[sys_.vv_of_cpl][:, fes.dof_vbar.is_free][sys_.free_cpl].tocsr()


def coarse_matrix(fes, nu, penalty_C=4.0):
    """P1 strain form + Gamma_Ntilde tangential penalty on free dofs;
    `preconditioners.py:121-165`."""
    m, k = fes.mesh, fes.k
    dl = np.array([[-1.0, -1.0], [1.0, 0.0], [0.0, 1.0]])
    rows, cols, vals = [], [], []
    for t in range(m.num_triangles):
        dlam = dl @ fes.Jinv[t]
        eps = np.zeros((6, 2, 2))
        for lv in range(3):
            for c in range(2):
                g = np.zeros((2, 2))
                g[c] = dlam[lv]
                eps[2 * lv + c] = 0.5 * (g + g.T)
        blk = nu * 0.5 * fes.detJ[t] * np.einsum("aij,bij->ab", eps, eps)
        lg = fes.dof_vbar.loc2glob[t]
        rows.append(np.repeat(lg, 6)); cols.append(np.tile(lg, 6)); vals.append(blk.ravel())
    if penalty_C > 0:
        mass = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
        for f in sorted(fes.regions.tilde_neumann_facets):
            a = m.facet_start[f]
            b = m.facets[f, 0] if m.facets[f, 0] != a else m.facets[f, 1]
            tF, ln = m.facet_tangent[f], m.facet_length[f]
            wgt = nu * penalty_C * k * k / ln
            dofs = np.array([2 * a, 2 * a + 1, 2 * b, 2 * b + 1])
            blk = np.zeros((4, 4))
            for i in range(2):
                for j in range(2):
                    blk[2 * i:2 * i + 2, 2 * j:2 * j + 2] = wgt * ln * mass[i, j] * np.outer(tF, tF)
            rows.append(np.repeat(dofs, 4)); cols.append(np.tile(dofs, 4)); vals.append(blk.ravel())
    n = fes.dof_vbar.ndof
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    free = fes.dof_vbar.is_free
    return A[free][:, free].tocsc()


class Asp:
    """`AspPreconditioner` (`preconditioners.py:286-336`) with the Jacobi
    smoother and an exact SuperLU coarse solve (`:165-171`)."""

    def __init__(self, A, jac, E, C, mode):
        if mode not in ("additive", "multiplicative"):
            raise ValueError(f"unknown composition mode {mode!r}")
        self.A, self.jac, self.E, self.mode = A, jac, E, mode
        self.lu = spla.splu(C)
        self.scale = 1.0
        if mode == "multiplicative":                               # :304-314
            rng = np.random.default_rng(1234)
            x = rng.standard_normal(A.shape[0])
            lam = 1.0
            for _ in range(20):
                y = jac.apply(A @ x)
                lam = np.linalg.norm(y)
                x = y / lam
            self.scale = 1.1 * lam

    def coarse(self, r):
        return self.E @ self.lu.solve(self.E.T @ r)

    def apply(self, r):
        if self.mode == "additive":
            return self.jac.apply(r) + self.coarse(r)
        x = np.zeros_like(r)
        x += self.jac.apply(r - self.A @ x) / self.scale
        x += self.coarse(r - self.A @ x)
        x += self.jac.apply(r - self.A @ x) / self.scale
        return x


class ExtendedAsp:
    """`preconditioners.py:353-378`."""

    def __init__(self, sys_, inner):
        self.s, self.inner = sys_, inner

    def apply(self, r_free):
        s = self.s
        fes = s.fes
        r = np.zeros(fes.n_vv)
        r[s.free_vv] = r_free
        w = r.copy()
        bubble = []
        for t in range(fes.mesh.num_triangles):
            r_o = r[s.l2g[t][s.iint]]
            bubble.append(sla.cho_solve(s.chol[t], r_o, check_finite=False))
            np.subtract.at(w, s.l2g[t][s.icpl], (s.X[t].T @ r_o) * s.sg[t][s.icpl])
        z = self.inner.apply(w[s.vv_of_cpl][s.free_cpl])
        out = np.zeros(fes.n_vv)
        zc = np.zeros(len(s.vv_of_cpl))
        zc[s.free_cpl] = z
        out[s.vv_of_cpl] = zc
        for t in range(fes.mesh.num_triangles):
            loc = out[s.l2g[t][s.icpl]] * s.sg[t][s.icpl]
            out[s.l2g[t][s.iint]] = bubble[t] - s.X[t] @ loc
        return out[s.free_vv]


def build_preconditioner(fes, sys_, nu, composition, penalty_C=4.0):
    """`driver.py:94-101` with smoother="jacobi"."""
    A = sys_.Sd_free()
    jac = Jacobi(A, facet_blocks_schur(fes, sys_))
    asp = Asp(A, jac, embedding_cpl(fes, sys_), coarse_matrix(fes, nu, penalty_C),
              composition)
    return ExtendedAsp(sys_, asp), asp


def cg(apply_A, b, apply_M, rtol=1e-8, maxit=1000):
    """`krylov.py:103-137`; returns (x, iterations, residual history)."""
    b = np.asarray(b, dtype=float)
    x = np.zeros_like(b)
    r = b.copy()
    bn = np.linalg.norm(b)
    res = [1.0]
    if bn == 0:
        return x, 0, res
    z = apply_M(r)
    p = z.copy()
    rz = r @ z
    it = 0
    for it in range(1, maxit + 1):
        Ap = apply_A(p)
        pAp = p @ Ap
        if pAp <= 0:
            raise NegativeCurvatureError(f"p'Ap = {pAp:.3e} at iteration {it}")
        a = rz / pAp
        x += a * p
        r -= a * Ap
        res.append(np.linalg.norm(r) / bn)
        if res[-1] <= rtol:
            break
        z = apply_M(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, it, res


# ------------------------------------------------------------ Stokes mode


def assemble_B(fes, bpu):
    """Pressure rows over all (V, Vhat) dofs; `condensation.py:178-186`
    (bpu per element, signs of the V dofs)."""
    l2g, sg = vv_maps(fes)
    nu_l = fes.bdm.ndof
    nt = fes.mesh.num_triangles
    vals = np.broadcast_to(bpu[None], (nt,) + bpu.shape) * sg[:, None, :nu_l]
    rows = np.repeat(fes.dof_q.loc2glob, nu_l, axis=1).ravel()
    cols = np.tile(l2g[:, :nu_l], (1, bpu.shape[0])).ravel()
    return sp.coo_matrix((vals.ravel(), (rows, cols)),
                         shape=(fes.dof_q.ndof, fes.n_vv)).tocsr()


def pressure_mass_diag(fes, nu):
    """`preconditioners.py:390-396`: detJ_t / nu on the element's dofs."""
    d = np.empty(fes.dof_q.ndof)
    for t in range(fes.mesh.num_triangles):
        d[fes.dof_q.loc2glob[t]] = fes.detJ[t] / nu
    return d


def saddle_apply(velocity_apply, diag, B_free):
    """`preconditioners.py:405-420`."""
    def apply(r):
        nv = B_free.shape[1]
        r_u, r_p = r[:nv], r[nv:]
        a = velocity_apply(r_u)
        dp = (r_p - B_free @ a) / diag
        du = a - velocity_apply(B_free.T @ dp)
        return np.concatenate([du, dp])
    return apply


def gmres(apply_A, b, apply_M=None, rtol=1e-6, maxit=500, project=None):
    """`krylov.py:25-100` (full GMRES, right preconditioned, modified
    Gram-Schmidt, Givens rotations); returns (x, iterations, residuals)."""
    if apply_M is None:
        apply_M = lambda v: v
    b = np.asarray(b, dtype=float)
    if project is not None:
        b = project(b)
    n = len(b)
    r0 = b.copy()
    beta = np.linalg.norm(r0)
    bnorm = np.linalg.norm(b)
    res = [1.0 if bnorm == 0 else beta / bnorm]
    if bnorm == 0.0 or beta / bnorm <= rtol:
        return np.zeros(n), 0, res
    V = [r0 / beta]
    H = np.zeros((maxit + 1, maxit))
    cs, sn = np.zeros(maxit), np.zeros(maxit)
    g = np.zeros(maxit + 1)
    g[0] = beta
    j = 0
    while j < maxit:
        w = np.array(apply_A(apply_M(V[j])), dtype=float)
        if project is not None:
            w = project(w)
        for i in range(j + 1):
            H[i, j] = w @ V[i]
            w -= H[i, j] * V[i]
        H[j + 1, j] = np.linalg.norm(w)
        for i in range(j):
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        hsub = H[j + 1, j]
        denom = np.hypot(H[j, j], hsub)
        cs[j], sn[j] = H[j, j] / denom, hsub / denom
        H[j, j], H[j + 1, j] = denom, 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        res.append(abs(g[j + 1]) / bnorm)
        happy = hsub <= 1e-14 * denom
        if not happy:
            V.append(w / hsub)
        j += 1
        if res[-1] <= rtol or happy:
            break
    y = np.linalg.solve(H[:j, :j], g[:j])
    x = apply_M(np.array(V[:j]).T @ y)
    if project is not None:
        x = project(x)
    return x, j, res


# ------------------------------------------------------------- post checks


def post_checks(fes, u, sigma, residuals):
    """`driver.py:183-218` (pointwise divergence over the H1 seminorm,
    nt-jump of the stress across interior facets, residual monotonicity),
    restated on this package's FeSystem tables (the same formulas as
    assembly.py:362-387)."""
    max_div, grad_scale = 0.0, 0.0
    for t in range(fes.mesh.num_triangles):
        uloc = u[fes.dof_v.loc2glob[t]] * fes.dof_v.signs[t]
        max_div = max(max_div, float(np.abs(uloc @ fes.tab_u_div / fes.detJ[t]).max()))
        grad = np.einsum("ia,upab,bj->upij", fes.J[t], fes.tab_u_grad, fes.Jinv[t]) / fes.detJ[t]
        g = np.einsum("u,upij->pij", uloc, grad)
        wq = fes.quad_tri.weights * fes.detJ[t]
        grad_scale += float(np.einsum("pij,p->", g * g, wq))
    grad_scale = max(1.0, np.sqrt(grad_scale))
    jump_max, scale = 0.0, 1e-300
    for f in fes.mesh.interior_facets:
        vals = []
        for t in fes.mesh.facet_tri[f]:
            le = int(np.nonzero(fes.edge_facet[t] == f)[0][0])
            sloc = sigma[fes.dof_sigma.loc2glob[t]] * fes.dof_sigma.signs[t]
            sv = np.einsum("s,spij->pij", sloc, fes.map_stress(t, fes.tab_sigma_edge[:, le]))
            nt = np.einsum("i,pij,j->p", fes.mesh.facet_tangent[f], sv, fes.mesh.facet_normal[f])
            if fes.edge_flip[t, le]:
                nt = nt[::-1]
            vals.append(nt)
        jump_max = max(jump_max, float(np.abs(vals[0] - vals[1]).max()))
        scale = max(scale, float(np.abs(vals[0]).max()))
    res = residuals
    monotone = all(res[i + 1] <= res[i] * (1 + 1e-12) for i in range(len(res) - 1))
    return {"max_div_scaled": max_div / grad_scale,
            "nt_jump_scaled": jump_max / max(scale, 1.0), "residual_monotone": monotone}


# -------------------------------------------------------------- microbench


def spd_schur(A, B):
    """S = B^T A^-1 B by the reference idiom cho_factor / cho_solve / B^T X
    (`condensation.py:216-224`)."""
    ch = sla.cho_factor(A, check_finite=False)
    return B.T @ sla.cho_solve(ch, B, check_finite=False)


def microbench_inputs(count, n=60, m=36, seed=3, chunk=65536):
    """BASELINE config 5 stream: per chunk G ~ N(0,1)^(c,n,n)
    then B ~ N(0,1)^(c,n,m) from default_rng(seed); A = G G^T + n I."""
    rng = np.random.default_rng(seed)
    As, Bs, done = [], [], 0
    while done < count:
        c = min(chunk, count - done)
        G = rng.standard_normal((c, n, n))
        B = rng.standard_normal((c, n, m))
        As.append(G @ np.swapaxes(G, 1, 2) + n * np.eye(n))
        Bs.append(B)
        done += c
    return np.concatenate(As), np.concatenate(Bs)
