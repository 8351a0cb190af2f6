"""Drop-in auxiliary-space preconditioner for the condensed velocity block.

Reference: `preconditioners.py:27-378` with `driver.py:82-102`.  The GPU path
covers the north-star configuration: target "Sd", smoother "jacobi",
composition "additive" or "multiplicative" (any `steps`).  Gauss-Seidel and
l1 are sequential / out of scope and are rejected with the
reference's exception types.

Per application everything runs in CUDA kernels on free-dof vectors:
  ExtendedAsp   mcs_ext_restrict -> mcs_gather_sub -> inner -> mcs_scatter
                -> mcs_ext_prolong                                   (A8)
  Jacobi        mcs_jacobi_apply over SoA packed facet-block inverses (A9)
  E_c, E_c^T    mcs_csr_spmv (transpose stored explicitly)           (A10)
  coarse        exact: dense inverse (small) or multifrontal (A11)
  S_d apply     mcs_apply_elem (multiplicative composition)          (A6)
Host work is setup only (index maps, E_c, the P1 coarse matrix and its
exact factorisation).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import List

import numpy as np
import scipy.sparse as sp

from . import _abi, engine
from .basis import shifted_legendre
from .coarse import CoarseSolver, factorize_coarse
from .maps import facet_slots, free_index
from .operators import SdOperator, as_device, axpby, empty, workspace


# ----------------------------------------------------------------- embedding

def _facet_moments(fes):
    """m[iv, q] = int_0^1 hat_iv L_q over the edge rule (hat_0 = 1-s)."""
    qe = fes.quad_edge
    leg = shifted_legendre(fes.k, qe.points)
    hat = np.vstack([1.0 - qe.points, qe.points])
    return np.array([[np.sum(qe.weights * hat[iv] * leg[q]) for q in range(fes.k + 1)]
                     for iv in range(2)])


def embedding_facet_coo(fes):
    """Facet rows of E (reference `preconditioners.py:40-63`), vectorised:
    V normal moments |F| m[iv,q] n_F[c] and Vhat tangential moments
    m[iv,q] t_F[c] (zero rows on Gamma_Ntilde)."""
    m, k = fes.mesh, fes.k
    nf = m.num_facets
    mom = _facet_moments(fes)
    ends = np.stack([m.facet_start, m.facet_end()], axis=1)       # (nf, 2)
    rows, cols, vals = [], [], []
    F = np.arange(nf)
    for iv in range(2):
        for q in range(k + 1):
            mv = m.facet_length * mom[iv, q]
            keep = np.abs(mv) >= 1e-15
            for c in range(2):
                rows.append(F[keep] * (k + 1) + q)
                cols.append(2 * ends[keep, iv] + c)
                vals.append(mv[keep] * m.facet_normal[keep, c])
        tilde = np.zeros(nf, dtype=bool)
        tilde[list(fes.regions.tilde_neumann_facets)] = True
        for q in range(k):
            if abs(mom[iv, q]) < 1e-15:
                continue
            keep = ~tilde
            for c in range(2):
                rows.append(fes.n_v + F[keep] * k + q)
                cols.append(2 * ends[keep, iv] + c)
                vals.append(mom[iv, q] * m.facet_tangent[keep, c])
    return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def _interior_coo(fes, Ef):
    """Interior bubble rows of E (reference `preconditioners.py:66-91`):
    per element the L2 fit of the P1 field against the facet part,
    vectorised over elements with batched solves."""
    k = fes.k
    n_em, n_int = 3 * (k + 1), (k + 1) * (k - 1)
    w = fes.quad_tri.weights
    U = fes.tab_u                                                 # (nu, nq, 2)
    JtJ = np.einsum("tci,tcj->tij", fes.J, fes.J)
    G = np.einsum("upi,p,vpj->ijuv", U, w, U)                     # (2,2,nu,nu)
    gram = np.einsum("tij,ijuv->tuv", JtJ, G) / fes.detJ[:, None, None]
    lam = np.stack([1 - fes.quad_tri.points[:, 0] - fes.quad_tri.points[:, 1],
                    fes.quad_tri.points[:, 0], fes.quad_tri.points[:, 1]])
    Mref = np.einsum("upj,p,lp->ulj", U[n_em:], w, lam)            # (n_int,3,2)
    mom = np.einsum("tcj,ulj->tulc", fes.J, Mref)                 # (nt,n_int,3,2)
    lg = fes.dof_v.loc2glob[:, :n_em]
    sg = fes.dof_v.signs[:, :n_em]
    tri = fes.mesh.triangles
    nt = len(tri)
    rows, cols, vals = [], [], []
    gii, gie = gram[:, n_em:, n_em:], gram[:, n_em:, :n_em]
    for lv in range(3):
        v = tri[:, lv]
        for c in range(2):
            col = 2 * v + c
            ced = np.asarray(Ef[lg.ravel(), np.repeat(col, n_em)]).reshape(nt, n_em) * sg
            rhs = mom[:, :, lv, c] - np.einsum("tie,te->ti", gie, ced)
            cint = np.linalg.solve(gii, rhs[:, :, None])[:, :, 0]
            keep = np.abs(cint) > 1e-14
            tt, ii = np.nonzero(keep)
            rows.append(fes.dof_v.loc2glob[tt, n_em + ii])
            cols.append(col[tt])
            vals.append(cint[keep])
    return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def build_embedding(fes, interior: bool = True) -> sp.csr_matrix:
    """E: Vbar -> (V, Vhat) (reference `preconditioners.py:27-94`)."""
    r, c, v = embedding_facet_coo(fes)
    shape = (fes.n_vv, fes.dof_vbar.ndof)
    Ef = sp.coo_matrix((v, (r, c)), shape=shape).tocsr()
    if not interior:
        return Ef
    ri, ci, vi = _interior_coo(fes, Ef)
    return sp.coo_matrix((np.concatenate([v, vi]), (np.concatenate([r, ri]),
                          np.concatenate([c, ci]))), shape=shape).tocsr()


def embedding_free(fes, E):
    return E[fes.vv_free][:, fes.dof_vbar.is_free].tocsr()


def embedding_cpl(fes, sys, E=None) -> sp.csr_matrix:
    """E restricted to free coupling rows and free P1 columns
    (reference `preconditioners.py:101-105`).  Only facet rows survive, so
    E may be the facet-only embedding."""
    if E is None:
        E = build_embedding(fes, interior=False)
    free_cpl = sys.free_mask_cpl()
    return E[sys.vv_of_cpl][:, fes.dof_vbar.is_free][free_cpl].tocsr()


# -------------------------------------------------------------- coarse space

def coarse_matrix(fes, nu, penalty_C=4.0):
    """Conforming P1 strain form + Gamma_Ntilde tangential penalty on free
    P1 dofs (reference `preconditioners.py:121-165`), vectorised."""
    m, k = fes.mesh, fes.k
    dl = np.array([[-1.0, -1.0], [1.0, 0.0], [0.0, 1.0]])
    dlam = np.einsum("la,tab->tlb", dl, fes.Jinv)                  # (nt,3,2)
    nt = m.num_triangles
    g = np.zeros((nt, 6, 2, 2))
    for lv in range(3):
        for c in range(2):
            g[:, 2 * lv + c, c, :] = dlam[:, lv]
    eps = 0.5 * (g + np.swapaxes(g, 2, 3))
    blk = nu * (0.5 * fes.detJ)[:, None, None] * np.einsum("taij,tbij->tab", eps, eps)
    lg = fes.dof_vbar.loc2glob
    rows = [np.repeat(lg, 6, axis=1).ravel()]
    cols = [np.tile(lg, (1, 6)).ravel()]
    vals = [blk.ravel()]
    if penalty_C > 0 and fes.regions.tilde_neumann_facets:
        Fs = np.array(sorted(fes.regions.tilde_neumann_facets))
        a, b = m.facet_start[Fs], m.facet_end()[Fs]
        tF, ln = m.facet_tangent[Fs], m.facet_length[Fs]
        wgt = nu * penalty_C * k * k / ln
        mass = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
        dofs = np.stack([2 * a, 2 * a + 1, 2 * b, 2 * b + 1], axis=1)
        tt = np.einsum("fi,fj->fij", tF, tF)
        B = np.zeros((len(Fs), 4, 4))
        for i in range(2):
            for j in range(2):
                B[:, 2 * i:2 * i + 2, 2 * j:2 * j + 2] = \
                    (wgt * ln * mass[i, j])[:, None, None] * tt
        rows.append(np.repeat(dofs, 4, axis=1).ravel())
        cols.append(np.tile(dofs, (1, 4)).ravel())
        vals.append(B.ravel())
    n = fes.dof_vbar.ndof
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    free = fes.dof_vbar.is_free
    return A[free][:, free].tocsr()


def build_coarse(fes, nu: float, penalty_C: float = 4.0, scale: float = 1.0) -> CoarseSolver:
    """Exactly factorised P1 coarse problem (reference `:121-171`)."""
    A = coarse_matrix(fes, nu, penalty_C)
    xy = fes.mesh.vertices[np.flatnonzero(fes.dof_vbar.is_free) // 2]
    return factorize_coarse(A, xy, scale=scale)


# ------------------------------------------------------------------ smoother

def facet_blocks_schur(fes, sys) -> List[np.ndarray]:
    """Host list of the S_d facet blocks (reference `:266-280`), for
    compatibility; the GPU smoother builds its blocks from `facet_slots`."""
    k = fes.k
    idx = free_index(sys.free_mask_cpl())
    out = []
    for f in range(fes.mesh.num_facets):
        d = [sys.cpl_of_vv[f * (k + 1) + q] for q in range(k + 1)]
        d += [sys.cpl_of_vv[fes.n_v + f * k + q] for q in range(k)]
        b = idx[np.array(d)]
        b = b[b >= 0]
        if len(b):
            out.append(np.unique(b))
    return out


class FacetBlockSmoother:
    """Facet-block Jacobi with packed block inverses in HBM (reference
    `preconditioners.py:177-206`, variant "jacobi").

    * `A` an `SdOperator` and `blocks` None (the driver path): the facet
      blocks of `facet_blocks_schur` are assembled on the GPU from the
      per-element Sd_T and inverted there (`mcs_jacobi_setup`).
    * `A` a SciPy sparse matrix (or an `SdOperator` with an explicit block
      list), as the reference takes it: the dense blocks A[blk, blk] are
      gathered on the host and inverted on the GPU (`mcs_block_inverse`);
      blocks must be disjoint (x[blk] = A_bb^-1 r[blk], like the reference's
      `jacobi_apply` for the S_d blocks) and hold at most 13 dofs.
    Gauss-Seidel and l1 are sequential over facets and out of the GPU scope
    (SURVEY §2): NotImplementedError; unknown variants: ValueError."""

    def __init__(self, A, blocks=None, variant: str = "gauss_seidel", factors=None):
        # `factors` mirrors the reference dataclass field; the GPU keeps packed
        # inverses instead (self.binv) and ignores it
        if variant not in ("jacobi", "gauss_seidel", "l1"):
            raise ValueError(f"unknown smoother variant {variant!r}")
        if variant != "jacobi":
            raise NotImplementedError(
                f"smoother {variant!r} is sequential / out of the GPU scope (SURVEY §2)")
        self.A, self.variant, self.blocks = A, variant, blocks
        if isinstance(A, SdOperator) and blocks is None:
            self._setup_from_sd(A)
        else:
            Ah = A.sys.Sd[A.sys.free_mask_cpl()][:, A.sys.free_mask_cpl()] \
                if isinstance(A, SdOperator) else A
            if not sp.issparse(Ah):
                raise TypeError("FacetBlockSmoother needs an SdOperator or a sparse matrix")
            if blocks is None:
                raise ValueError("a sparse matrix needs its block list")
            self._setup_from_blocks(sp.csr_matrix(Ah), blocks)

    def _setup_from_sd(self, A):
        torch = __import__("torch")
        sys_ = A.sys
        fes = sys_.fes
        k = fes.k
        slots, self.facets = facet_slots(fes, sys_.maps)
        self.nblk = len(slots)
        B = 2 * k + 1
        self.binv = torch.empty((B * (B + 1) // 2, self.nblk), dtype=torch.float64, device="cuda")
        self.bidx = torch.empty((B, self.nblk), dtype=torch.int32, device="cuda")
        self.bsize = torch.empty(self.nblk, dtype=torch.int32, device="cuda")
        info = torch.empty(self.nblk, dtype=torch.int32, device="cuda")
        m = sys_.dev_maps()
        slots_d = engine.to_dev(slots)              # alive until the kernel has run
        _abi.call("mcs_jacobi_setup", k, self.nblk, _abi.ptr(sys_.Sd_dev),
                  sys_.Sd_dev.shape[1], _abi.ptr(m["cpl_codes"]),
                  _abi.ptr(slots_d), _abi.ptr(self.binv), _abi.ptr(self.bidx),
                  _abi.ptr(self.bsize), _abi.ptr(info), _abi.stream())
        bad = np.flatnonzero(info.cpu().numpy())
        if len(bad):
            raise RuntimeError(f"facet block {int(self.facets[bad[0]])} not SPD")
        self.k = k

    def _setup_from_blocks(self, A, blocks):
        torch = __import__("torch")
        sizes = np.array([len(b) for b in blocks], dtype=np.int32)
        if len(blocks) == 0:
            raise ValueError("empty block list")
        bmax = int(sizes.max())
        if bmax > 13:
            raise NotImplementedError(f"facet blocks of {bmax} > 13 dofs (k > 6)")
        k = max(2, bmax // 2)                          # template block size 2k+1 >= bmax
        B = 2 * k + 1
        nblk = len(blocks)
        idx = np.full((nblk, B), -1, dtype=np.int64)
        for i, b in enumerate(blocks):
            idx[i, :len(b)] = b
        covered = idx[idx >= 0]
        if len(np.unique(covered)) != len(covered):
            raise NotImplementedError("overlapping smoother blocks (only disjoint facet blocks)")
        ii = np.repeat(idx, B, axis=1).ravel()
        jj = np.tile(idx, (1, B)).ravel()
        ok = (ii >= 0) & (jj >= 0)
        dense = np.zeros(nblk * B * B)
        dense[ok] = np.asarray(A[ii[ok], jj[ok]]).ravel()
        self.nblk, self.k, self.facets = nblk, k, np.arange(nblk)
        self.binv = torch.empty((B * (B + 1) // 2, nblk), dtype=torch.float64, device="cuda")
        self.bidx = torch.empty((B, nblk), dtype=torch.int32, device="cuda")
        self.bsize = engine.to_dev(sizes)
        info = torch.empty(nblk, dtype=torch.int32, device="cuda")
        dense_d, idx_d = engine.to_dev(dense), engine.to_dev(idx.astype(np.int32))
        _abi.call("mcs_block_inverse", k, nblk, _abi.ptr(dense_d), _abi.ptr(idx_d),
                  _abi.ptr(self.bsize), _abi.ptr(self.binv), _abi.ptr(self.bidx),
                  _abi.ptr(info), _abi.stream())
        bad = np.flatnonzero(info.cpu().numpy())
        if len(bad):
            raise RuntimeError(f"smoother block {int(bad[0])} not SPD")

    @_abi.nvtx("facet_jacobi")
    def jacobi_apply(self, r, out=None, scale_inv=1.0, stream=None):
        rd, host = as_device(r)
        x = out if out is not None else empty(rd.numel())
        if self.blocks is not None:              # caller blocks need not cover every dof
            x.zero_()
        _abi.call("mcs_jacobi_apply", self.k, self.nblk, _abi.ptr(self.binv),
                  _abi.ptr(self.bidx), _abi.ptr(rd), _abi.ptr(x), float(scale_inv),
                  _abi.stream(stream))
        return x.cpu().numpy() if host else x

    apply_symmetric = jacobi_apply


class _DevCsr:
    def __init__(self, A: sp.csr_matrix):
        A = A.tocsr()
        A.sort_indices()
        self.shape = A.shape
        self.ptr = engine.to_dev(A.indptr.astype(np.int32))
        self.col = engine.to_dev(A.indices.astype(np.int32))
        self.val = engine.to_dev(A.data.astype(np.float64))
        avg = A.nnz / max(A.shape[0], 1)
        self.lanes = 1 if avg <= 6 else (4 if avg <= 16 else 8)

    def mv(self, x, y, alpha=1.0, beta=0.0, stream=None):
        _abi.call("mcs_csr_spmv", self.shape[0], _abi.ptr(self.ptr), _abi.ptr(self.col),
                  _abi.ptr(self.val), _abi.ptr(x), _abi.ptr(y), float(alpha), float(beta),
                  self.lanes, _abi.stream(stream))
        return y


class _CsrOperator:
    """A SciPy CSR matrix applied on the GPU (`mcs_csr_spmv`)."""

    graphable = True

    def __init__(self, A):
        self.M = _DevCsr(A)
        self.shape = A.shape

    def apply(self, x, out=None, stream=None):
        xd, host = as_device(x)
        y = out if out is not None else empty(self.shape[0])
        self.M.mv(xd, y, 1.0, 0.0, stream)
        return y.cpu().numpy() if host else y

    __call__ = apply


# MCS_NO_FORK=1: A/B switch, additive ASP smoother and coarse chain in one stream
FORK_ADDITIVE = os.environ.get("MCS_NO_FORK", "0") != "1"


class AspPreconditioner:
    """Smoother + embedded exact coarse correction (reference `:286-336`)."""

    def __init__(self, A, smoother, E, coarse, mode: str = "multiplicative",
                 steps: int = 1):
        """`A` is an `SdOperator` or, as in the reference, a SciPy sparse
        matrix (applied on the GPU as a CSR); `coarse` is this package's
        `CoarseSolver` or the reference's (its `matrix` is refactorised
        exactly for the GPU)."""
        if mode not in ("additive", "multiplicative"):
            raise ValueError(f"unknown composition mode {mode!r}")
        if sp.issparse(A):
            A = _CsrOperator(A)
        if not hasattr(coarse, "solve_dev"):
            coarse = factorize_coarse(sp.csr_matrix(coarse.matrix), None,
                                      scale=getattr(coarse, "scale", 1.0))
        self.A, self.smoother, self.coarse, self.mode, self.steps = A, smoother, coarse, mode, steps
        self.E = _DevCsr(E)
        self.Et = _DevCsr(E.T.tocsr())
        n, nc = E.shape
        self.n = n
        self._t, self._w = empty(n), empty(n)
        self._u, self._v = empty(nc), empty(nc)
        self._side = self._ev = None
        self.jacobi_scale = 1.0
        if mode == "multiplicative":
            self.jacobi_scale = self._estimate_smoother_bound()

    def _estimate_smoother_bound(self, iters=20, seed=1234):
        """1.1 x the largest Ritz value of J A by 20 power steps from
        default_rng(1234) (reference `:304-314`), on the GPU."""
        ws = workspace()
        x = as_device(np.random.default_rng(seed).standard_normal(self.n))[0]
        y = empty(self.n)
        lam = 1.0
        for _ in range(iters):
            self.A.apply(x, out=self._t)
            self.smoother.jacobi_apply(self._t, out=y)
            lam = float(np.sqrt(ws.dot_host(y, y)))
            axpby(1.0 / lam, y, 0.0, x)
        return 1.1 * lam

    @_abi.nvtx("coarse_correction")
    def coarse_correction(self, r, x, beta):
        """x = beta*x + E C^-1 E^T r."""
        self.Et.mv(r, self._u)
        self.coarse.solve_dev(self._u, self._v)
        self.E.mv(self._v, x, 1.0, beta)
        return x

    def apply(self, r, out=None):
        rd, host = as_device(r)
        x = out if out is not None else empty(self.n)
        if self.mode == "additive" and FORK_ADDITIVE:
            # the smoother and the coarse chain are independent until the
            # final x += E v: the smoother runs on a side stream (a graph
            # branch under capture) while E^T r and the coarse solve run here
            torch = __import__("torch")
            main = torch.cuda.current_stream()
            if self._side is None:
                self._side = torch.cuda.Stream()
                self._ev = (torch.cuda.Event(), torch.cuda.Event())
            self._ev[0].record(main)
            self._side.wait_event(self._ev[0])
            self.smoother.jacobi_apply(rd, out=x, stream=self._side)
            self._ev[1].record(self._side)
            self.Et.mv(rd, self._u)
            self.coarse.solve_dev(self._u, self._v)
            main.wait_event(self._ev[1])
            self.E.mv(self._v, x, 1.0, 1.0)
        elif self.mode == "additive":
            self.smoother.jacobi_apply(rd, out=x)
            self.coarse_correction(rd, x, 1.0)
        else:
            s_inv = 1.0 / self.jacobi_scale
            t, w = self._t, self._w
            # pre-smoothing: first step has x = 0, so r - A x = r exactly
            self.smoother.jacobi_apply(rd, out=x, scale_inv=s_inv)
            for _ in range(self.steps - 1):
                self._residual(rd, x, t)
                self.smoother.jacobi_apply(t, out=w, scale_inv=s_inv)
                axpby(1.0, w, 1.0, x)
            self._residual(rd, x, t)
            self.coarse_correction(t, x, 1.0)
            for _ in range(self.steps):
                self._residual(rd, x, t)
                self.smoother.jacobi_apply(t, out=w, scale_inv=s_inv)
                axpby(1.0, w, 1.0, x)
        return x.cpu().numpy() if host else x

    def _residual(self, r, x, t):
        self.A.apply(x, out=t)
        axpby(1.0, r, -1.0, t)


class ExtendedAsp:
    """S_d preconditioner lifted to S through the exact block factorisation
    (reference `:339-378`)."""

    graphable = True          # every stage is a stream-ordered kernel

    def __init__(self, sys, inner):
        if sys.Sd_dev is None:
            raise ValueError("double_schur() must be run first")
        self.sys, self.inner = sys, inner
        m = sys.maps
        self.n, self.nc = m.n_vv_free, m.n_cpl_free
        nt = sys.S_dev.shape[0]
        self.nt = nt
        self.bubble = empty(nt * sys.z["n_int"])
        self.acc, self.wc = empty(self.nc), empty(self.nc)
        self.zc = empty(self.nc)

    @_abi.nvtx("extended_asp")
    def apply(self, r_free, out=None, stream=None):
        s = self.sys
        rd, host = as_device(r_free)
        out = out if out is not None else empty(self.n)
        m = s.dev_maps()
        st = _abi.stream(stream)
        _abi.call("mcs_ext_restrict", s.k, self.nt, _abi.ptr(s.ext_dev), _abi.ptr(m["bubble_idx"]),
                  _abi.ptr(m["cpl_codes"]), _abi.ptr(rd), _abi.ptr(self.bubble),
                  _abi.ptr(self.acc), self.nc, st)
        _abi.call("mcs_gather_sub", self.nc, _abi.ptr(rd), _abi.ptr(m["c2v"]),
                  _abi.ptr(self.acc), _abi.ptr(self.wc), st)
        self.inner.apply(self.wc, out=self.zc)
        # bubble dofs = bubble - X z_c, coupling dofs = z_c (scatter fused in)
        _abi.call("mcs_ext_prolong", s.k, self.nt, _abi.ptr(s.ext_dev), _abi.ptr(m["bubble_idx"]),
                  _abi.ptr(m["cpl_codes"]), _abi.ptr(self.zc), _abi.ptr(self.bubble),
                  _abi.ptr(m["c2v"]), _abi.ptr(out), st)
        return out.cpu().numpy() if host else out

    __call__ = apply


# ------------------------------------------------------ Stokes (saddle) mode

class PressureMassPrecond:
    """Exact inverse of the nu^-1-scaled pressure mass matrix (reference
    `preconditioners.py:384-402`): diagonal detJ_t / nu on the element-major
    pressure dofs (orthonormal element bases)."""

    def __init__(self, diag):
        torch = __import__("torch")
        self.diag = np.asarray(diag, dtype=float)
        self.diag_dev = torch.from_numpy(self.diag).cuda()

    @classmethod
    def build(cls, fes, nu: float):
        nq = fes.dof_q.loc2glob.shape[1]
        d = np.empty(fes.dof_q.ndof)
        d[fes.dof_q.loc2glob.ravel()] = np.repeat(fes.detJ / nu, nq)
        return cls(d)

    def apply(self, r, out=None, stream=None):
        rd, host = as_device(r)
        out = out if out is not None else empty(len(self.diag))
        _abi.call("mcs_vdiv", len(self.diag), _abi.ptr(rd), _abi.ptr(self.diag_dev),
                  _abi.ptr(out), _abi.stream(stream))
        return out.cpu().numpy() if host else out

    def mass_matrix(self):
        return sp.diags(self.diag).tocsr()


class SaddlePreconditioner:
    """Block triangular preconditioner, two velocity solves per application
    (reference `preconditioners.py:405-420`):
        a = V r_u;  dp = P (r_p - B a);  du = a - V (B^T dp)."""

    def __init__(self, velocity_apply, pressure: PressureMassPrecond, B_free):
        B = B_free
        self.velocity_apply, self.pressure, self.B = velocity_apply, pressure, B
        self.n_v, self.n_p = B.n_v, B.n_p
        self._a, self._bt, self._v2 = empty(self.n_v), empty(self.n_v), empty(self.n_v)
        self._bp = empty(self.n_p)

    def _vel(self, r, out):
        if hasattr(self.velocity_apply, "apply"):
            return self.velocity_apply.apply(r, out=out)
        out.copy_(self.velocity_apply(r))
        return out

    def apply(self, r, out=None, stream=None):
        rd, host = as_device(r)
        out = out if out is not None else empty(self.n_v + self.n_p)
        a = self._vel(rd[:self.n_v], self._a)
        self.B.apply(a, out=self._bp, stream=stream)
        axpby(1.0, rd[self.n_v:], -1.0, self._bp, stream)          # r_p - B a
        dp = self.pressure.apply(self._bp, out=out[self.n_v:], stream=stream)
        self.B.apply_T(dp, out=self._bt, stream=stream)
        v2 = self._vel(self._bt, self._v2)
        out[:self.n_v].copy_(a)
        axpby(-1.0, v2, 1.0, out[:self.n_v], stream)              # a - V(B^T dp)
        return out.cpu().numpy() if host else out

    __call__ = apply
