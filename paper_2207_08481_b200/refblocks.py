"""Element blocks as weighted sums of reference-cell matrices (host setup).

On an affine triangle every block of `assemble_element_blocks`
(reference `assembly.py:49-91`) is a short linear combination of matrices
that live on the reference cell, with weights that depend only on the
element geometry (J, detJ, the outward edge normals and the facet frames):

  msig = detJ/nu * sum_{a<=b} G_ab(J) Msym^{ab}         G_ab = T_a : T_b
  bws  = detJ * sum_a kappa_a(J) W^a                    kappa_a = skew(T_a)
  bus  = Bvol + sum_{e,a} w^{bus}_{e,a} E^{e,a}         (edge term -<s_nn, u_n>)
  bhs  = sum_{e,a} w^{bhs}_{e,a} H^{e,a}                (rows of edge e only)
  adiv = nu/(2 detJ) * Adiv
  bpu  = Bpu                                            (J-invariant)

with T_a = J^-T D_a J^T the Piola image of the trace-free generator D_a
(`dofmap.py:265-267`) and u = J u_hat / detJ (`dofmap.py:261-263`).  The GPU
block kernel evaluates exactly these sums; this module builds the reference
matrices once per k, the per-element weight table (vectorised over
elements), and a sparse (entry -> weight, value) program the kernels walk.
Parity with the reference quadrature is ~1e-15 relative
(`tests/test_refblocks.py`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .basis import DEV_COMPONENTS

# weight table layout (per element)
W_MSIG, W_BWS, W_BUSE, W_BHS, W_ADIV, W_ONE = 0, 6, 9, 18, 27, 28
N_WEIGHTS = 30                      # 29 used, padded to an even count
_PAIRS = ((0, 0), (1, 1), (2, 2), (0, 1), (0, 2), (1, 2))


def local_sizes(k: int) -> dict:
    ns = 3 * (k + 1) * (k + 2) // 2 - 3
    nw = k * (k + 1) // 2
    nu = (k + 1) * (k + 2)
    nh = 3 * k
    n_int = (k + 1) * (k - 1)
    nloc = nu + nh
    return dict(k=k, ns=ns, nw=nw, nu=nu, nh=nh, nloc=nloc, n_int=n_int,
                ncpl=nloc - n_int, n_em=3 * (k + 1), nq=k * (k + 1) // 2)


@dataclass
class BlockRefs:
    """Reference-cell matrices of one degree k."""
    k: int
    msig: np.ndarray      # (6, ns, ns)
    bws: np.ndarray       # (3, nw, ns)
    bus_vol: np.ndarray   # (nu, ns)
    bus_edge: np.ndarray  # (3, 3, nu, ns)      [edge, a]
    bhs: np.ndarray       # (3, 3, k, ns)       [edge, a]
    adiv: np.ndarray      # (nu, nu)
    bpu: np.ndarray       # (nq, nu)
    u_tab: np.ndarray     # (nu, nq_tri, 2) reference BDM values (for the load)


def build_refs(fes) -> BlockRefs:
    k = fes.k
    w = fes.quad_tri.weights
    we = fes.quad_edge.weights
    c = fes.tab_sigma_comp                          # (ns, nq, 3)
    ce = fes.tab_sigma_edge_comp                    # (ns, 3, nqe, 3)
    M = np.einsum("spa,p,zpb->absz", c, w, c)       # (3, 3, ns, ns)
    msig = np.stack([M[a, b] if a == b else M[a, b] + M[b, a]
                     for a, b in _PAIRS])
    bws = np.einsum("wp,p,spa->aws", fes.tab_w, w, c)
    bus_vol = np.einsum("upi,p,spi->us", fes.tab_u, w, fes.tab_sigma_div)
    ue = fes.tab_u_edge                             # (nu, 3, nqe, 2)
    # u_n = (u_hat . J^T n_out) / detJ and J^T n_out = n_hat_e / |J^-T n_hat_e|,
    # so only the reference normal component of u_hat enters
    from .quadrature import REF_NORMALS
    un_hat = np.einsum("uepi,ei->uep", ue, REF_NORMALS)
    bus_edge = np.einsum("uep,p,sepa->eaus", un_hat, we, ce)
    leg = fes.tab_leg_edge[:k]
    bhs = np.einsum("hp,p,sepa->eahs", leg, we, ce)
    adiv = np.einsum("up,p,vp->uv", fes.tab_u_div, w, fes.tab_u_div)
    bpu = np.einsum("qp,p,up->qu", fes.tab_q, w, fes.tab_u_div)
    return BlockRefs(k, msig, bws, bus_vol, bus_edge, bhs, adiv, bpu,
                     fes.tab_u.copy())


def element_weights(fes, nu: float) -> np.ndarray:
    """(nt, N_WEIGHTS) geometry weights, vectorised over elements."""
    J, det = fes.J, fes.detJ
    JinvT = fes.JinvT
    T = np.einsum("til,alm,tjm->taij", JinvT, DEV_COMPONENTS, J)   # (nt,3,2,2)
    G = np.einsum("taij,tbij->tab", T, T)
    nt = len(det)
    W = np.zeros((nt, N_WEIGHTS))
    for r, (a, b) in enumerate(_PAIRS):
        W[:, W_MSIG + r] = det / nu * G[:, a, b]
    W[:, W_BWS:W_BWS + 3] = det[:, None] * 0.5 * (T[:, :, 1, 0] - T[:, :, 0, 1])
    n = fes.edge_normal_out                          # (nt, 3, 2)
    ln = fes.edge_len                                # (nt, 3)
    snn = np.einsum("tei,taij,tej->tea", n, T, n)    # (nt, 3, 3)
    from .quadrature import REF_NORMALS
    rho = np.linalg.norm(np.einsum("tji,ej->tei", fes.Jinv, REF_NORMALS), axis=2)  # |J^-T n_hat|
    we = -(ln / (det[:, None] * rho))[:, :, None] * snn      # (nt, e, a)
    W[:, W_BUSE:W_BUSE + 9] = we.reshape(nt, 9)
    nF = fes.mesh.facet_normal[fes.edge_facet]
    tF = fes.mesh.facet_tangent[fes.edge_facet]
    tsn = np.einsum("tei,taij,tej->tea", tF, T, nF)
    wh = -(fes.edge_sign * ln)[:, :, None] * tsn
    W[:, W_BHS:W_BHS + 9] = wh.reshape(nt, 9)
    W[:, W_ADIV] = 0.5 * nu / det
    W[:, W_ONE] = 1.0
    return W


def dense_blocks(refs: BlockRefs, W: np.ndarray):
    """Host evaluation of the weighted sums for a few elements (tests and the
    single-element drop-in); the batched path runs on the GPU."""
    k = refs.k
    msig = np.einsum("tr,rij->tij", W[:, W_MSIG:W_MSIG + 6], refs.msig)
    bws = np.einsum("ta,awj->twj", W[:, W_BWS:W_BWS + 3], refs.bws)
    bus = refs.bus_vol[None] + np.einsum(
        "tr,rus->tus", W[:, W_BUSE:W_BUSE + 9], refs.bus_edge.reshape(9, *refs.bus_vol.shape))
    wh = W[:, W_BHS:W_BHS + 9].reshape(-1, 3, 3)
    bhs = np.einsum("tea,eahs->tehs", wh, refs.bhs).reshape(len(W), 3 * k, -1)
    adiv = W[:, W_ADIV, None, None] * refs.adiv[None]
    return msig, bws, bus, bhs, adiv


def load_vectors(fes, refs: BlockRefs, body_force) -> np.ndarray:
    """(nt, nu) element load vectors  sum_p w_p u_hat(p) . (J^T f(x_p))."""
    nt = fes.mesh.num_triangles
    nu_loc = refs.bus_vol.shape[0]
    if body_force is None:
        return np.zeros((nt, nu_loc))
    X = fes.phys_points()                            # (nt, nq, 2)
    vec = getattr(body_force, "vectorized", None)
    if vec is not None:
        F = np.asarray(vec(X.reshape(-1, 2)), dtype=float).reshape(X.shape)
    else:
        F = np.array([body_force(x) for x in X.reshape(-1, 2)],
                     dtype=float).reshape(X.shape)
    G = np.einsum("tji,tpj->tpi", fes.J, F) * fes.quad_tri.weights[None, :, None]
    return np.einsum("upi,tpi->tu", refs.u_tab, G)
