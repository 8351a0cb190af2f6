"""Global dof numbering, signs, constraints and element geometry (host setup).

`FeSystem` restates the reference `dofmap.py:53-276` with array operations
instead of per-element Python loops, keeping every numbering convention:

* V (BDM^k): facet normal moments `f*(k+1)+q`, then element bubbles
  `nf*(k+1) + t*n_int + i`; local order [edge-major facet dofs | bubbles];
  sign = (n_F . n_out) * (-1)^q if the facet parameter runs against the
  local edge (`dofmap.py:155-165`);
* Vhat: `f*k+q`, sign (-1)^q if flipped (`dofmap.py:174-183`);
* constraints: V on Gamma_D, Vhat on Gamma_D u Gamma_Ntilde, Vbar on the
  vertices of Gamma_D facets (`dofmap.py:166-211`).

The element geometry (J, detJ, outward edge normals, facet sign/flip) is what
the GPU block-generation weights are computed from.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import basis as fb
from .mesh import LOCAL_EDGES, BoundaryRegions, Mesh
from .quadrature import edge_points, edge_rule, triangle_rule


@dataclass
class SpaceDofMap:
    name: str
    ndof: int
    is_free: np.ndarray
    values: np.ndarray
    loc2glob: np.ndarray
    signs: np.ndarray

    @property
    def nfree(self):
        return int(self.is_free.sum())

    @property
    def free(self):
        return np.flatnonzero(self.is_free)

    def local_values(self, coeffs, t):
        return coeffs[self.loc2glob[t]] * self.signs[t]

    def full_vector(self, free_part):
        full = self.values.copy()
        full[self.is_free] = free_part
        return full


class _ScalarSpace:
    def __init__(self, k):
        self.degree, self.ndof = k, (k + 1) * (k + 2) // 2

    def eval(self, pts):
        return fb.scalar_pk_eval(self.degree, pts)

    eval_scalar = eval


class FeSystem:
    """Quadrature, reference tables, affine geometry and dof maps of one
    (mesh, boundary partition, k)."""

    def __init__(self, mesh: Mesh, regions: BoundaryRegions, k: int):
        if k < 2:
            raise ValueError(
                "degree k >= 2 required; the lowest-order variant is out of scope")
        self.mesh, self.regions, self.k = mesh, regions, k
        self.quad_tri = triangle_rule(2 * k + 2)
        self.quad_edge = edge_rule(2 * k + 2)
        self.bdm = fb.bdm_basis(k)
        self.sigma = fb.sigma_basis(k)
        self.skew = _ScalarSpace(k - 1)
        self.nq_loc = k * (k + 1) // 2
        self._geometry()
        self._tables()
        self._dofs()

    # ------------------------------------------------------------ geometry
    def _geometry(self):
        m = self.mesh
        P = m.vertices[m.triangles]                       # (nt, 3, 2)
        J = np.stack([P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]], axis=2)
        det = J[:, 0, 0] * J[:, 1, 1] - J[:, 0, 1] * J[:, 1, 0]
        Jinv = np.empty_like(J)
        Jinv[:, 0, 0] = J[:, 1, 1] / det
        Jinv[:, 0, 1] = -J[:, 0, 1] / det
        Jinv[:, 1, 0] = -J[:, 1, 0] / det
        Jinv[:, 1, 1] = J[:, 0, 0] / det
        self.J, self.detJ, self.Jinv = J, det, Jinv
        self.JinvT = np.swapaxes(Jinv, 1, 2)
        self.origin = P[:, 0]
        self.tri_diam = m.triangle_diameter()

        self.edge_facet = m.tri_facets
        A = m.triangles[:, LOCAL_EDGES[:, 0]]             # (nt, 3)
        B = m.triangles[:, LOCAL_EDGES[:, 1]]
        d = m.vertices[B] - m.vertices[A]                 # (nt, 3, 2)
        ln = np.linalg.norm(d, axis=2)
        n_out = np.stack([d[..., 1], -d[..., 0]], axis=2) / ln[..., None]
        mid = 0.5 * (m.vertices[A] + m.vertices[B])
        away = np.einsum("tei,tei->te", n_out, mid - P.mean(axis=1)[:, None, :])
        n_out = np.where((away < 0)[..., None], -n_out, n_out)
        self.edge_len = ln
        self.edge_normal_out = n_out
        nF = m.facet_normal[m.tri_facets]
        self.edge_sign = np.sign(np.einsum("tei,tei->te", n_out, nF))
        self.edge_flip = m.facet_start[m.tri_facets] != A

    # -------------------------------------------------------------- tables
    def _tables(self):
        k, qt, qe = self.k, self.quad_tri, self.quad_edge
        self.tab_sigma = self.sigma.eval(qt.points)             # (ns,nq,2,2)
        self.tab_sigma_comp = self.sigma.components(qt.points)  # (ns,nq,3)
        self.tab_sigma_div = self.sigma.div(qt.points)          # (ns,nq,2)
        self.tab_u, self.tab_u_grad = self.bdm.eval(qt.points, grad=True)
        self.tab_u_div = self.bdm.div(qt.points)                # (nu,nq)
        self.tab_w = self.skew.eval(qt.points)                  # (nw,nq)
        self.tab_q = fb.dubiner_eval(k - 1, qt.points)
        epts = [edge_points(e, qe.points) for e in range(3)]
        self.tab_sigma_edge = np.stack([self.sigma.eval(p) for p in epts], axis=1)
        self.tab_sigma_edge_comp = np.stack(
            [self.sigma.components(p) for p in epts], axis=1)   # (ns,3,nqe,3)
        self.tab_u_edge = np.stack([self.bdm.eval(p) for p in epts], axis=1)
        self.tab_leg_edge = fb.shifted_legendre(k, qe.points)

    # ---------------------------------------------------------------- dofs
    def _dofs(self):
        m, reg, k = self.mesh, self.regions, self.k
        nt, nf, nv = m.num_triangles, m.num_facets, m.num_vertices
        ne, n_int = k + 1, (k + 1) * (k - 1)
        fac = m.tri_facets                                   # (nt, 3)
        flip = self.edge_flip

        qn = np.arange(ne)
        l2g_f = (fac[:, :, None] * ne + qn).reshape(nt, 3 * ne)
        alt_n = np.where(flip[:, :, None], (-1.0) ** qn, 1.0)
        sg_f = (self.edge_sign[:, :, None] * alt_n).reshape(nt, 3 * ne)
        l2g_i = nf * ne + np.arange(nt)[:, None] * n_int + np.arange(n_int)
        nd_v = nf * ne + nt * n_int
        free_v = np.ones(nd_v, dtype=bool)
        dir_f = np.array(sorted(reg.dirichlet_facets), dtype=np.int64)
        if len(dir_f):
            free_v[(dir_f[:, None] * ne + qn).ravel()] = False
        self.dof_v = SpaceDofMap(
            "V", nd_v, free_v, np.zeros(nd_v), np.concatenate([l2g_f, l2g_i], 1),
            np.concatenate([sg_f, np.ones((nt, n_int))], 1))

        qh = np.arange(k)
        l2g_h = (fac[:, :, None] * k + qh).reshape(nt, 3 * k)
        sg_h = np.where(flip[:, :, None], (-1.0) ** qh, 1.0).reshape(nt, 3 * k)
        free_h = np.ones(nf * k, dtype=bool)
        con_h = np.array(sorted(reg.dirichlet_facets | reg.tilde_neumann_facets),
                         dtype=np.int64)
        if len(con_h):
            free_h[(con_h[:, None] * k + qh).ravel()] = False
        self.dof_vhat = SpaceDofMap("Vhat", nf * k, free_h, np.zeros(nf * k),
                                    l2g_h, sg_h)

        def local(name, n):
            return SpaceDofMap(name, nt * n, np.ones(nt * n, dtype=bool),
                               np.zeros(nt * n),
                               np.arange(nt)[:, None] * n + np.arange(n),
                               np.ones((nt, n)))

        self.dof_sigma = local("Sigma", self.sigma.ndof)
        self.dof_w = local("W", self.skew.ndof)
        self.dof_q = local("Q", self.nq_loc)

        l2g_b = (2 * m.triangles[:, :, None] + np.arange(2)).reshape(nt, 6)
        free_b = np.ones(2 * nv, dtype=bool)
        if len(dir_f):
            vd = m.facets[dir_f].ravel()
            free_b[2 * vd] = False
            free_b[2 * vd + 1] = False
        self.dof_vbar = SpaceDofMap("Vbar", 2 * nv, free_b, np.zeros(2 * nv),
                                    l2g_b, np.ones((nt, 6)))
        self._dirichlet_data()

        self.n_v, self.n_vhat = nd_v, nf * k
        self.n_vv = nd_v + nf * k
        self.vv_free = np.concatenate([free_v, free_h])
        self.vv_values = np.concatenate([self.dof_v.values, self.dof_vhat.values])
        interior = np.zeros(self.n_vv, dtype=bool)
        interior[nf * ne:nd_v] = True
        self.vv_interior = interior

    def _dirichlet_data(self):
        g = self.regions.dirichlet_value
        if g is None:
            return
        m, k, qe = self.mesh, self.k, self.quad_edge
        leg = fb.shifted_legendre(k, qe.points)
        end = m.facet_end()
        for f in sorted(self.regions.dirichlet_facets):
            pa, pb = m.vertices[m.facet_start[f]], m.vertices[end[f]]
            gv = np.array([g(pa + s * (pb - pa)) for s in qe.points])
            gn, gt = gv @ m.facet_normal[f], gv @ m.facet_tangent[f]
            self.dof_v.values[f * (k + 1):(f + 1) * (k + 1)] = \
                m.facet_length[f] * (leg @ (qe.weights * gn))
            self.dof_vhat.values[f * k:(f + 1) * k] = leg[:k] @ (qe.weights * gt)

    # ------------------------------------------------------------- helpers
    def map_vector(self, t, ref_vals):
        return np.einsum("ij,...j->...i", self.J[t], ref_vals) / self.detJ[t]

    def map_stress(self, t, ref_vals):
        return np.einsum("il,...lm,jm->...ij", self.JinvT[t], ref_vals, self.J[t])

    def phys_points(self, t=None):
        """Physical triangle quadrature points, (nq, 2) or (nt, nq, 2)."""
        if t is None:
            return self.origin[:, None, :] + np.einsum(
                "pj,tij->tpi", self.quad_tri.points, self.J)
        return self.origin[t] + self.quad_tri.points @ self.J[t].T

    def dof_counts(self):
        return {s.name: (s.ndof, s.nfree) for s in
                (self.dof_v, self.dof_vhat, self.dof_sigma, self.dof_w,
                 self.dof_q, self.dof_vbar)}


def build_dof_maps(mesh, regions, k) -> FeSystem:
    return FeSystem(mesh, regions, k)
