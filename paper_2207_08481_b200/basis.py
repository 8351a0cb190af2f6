"""Reference-cell polynomial bases (host setup, not on the GPU hot path).

The local bases define the meaning of every per-element matrix the GPU
kernels consume, so they are restated here with the same generators and the
same numerical recipe as the reference `basis.py`:

* orthonormal Dubiner scalars through the scaled Legendre / Jacobi
  recurrences (`basis.py:50-137`),
* the hierarchical scalar P^k used by the skew space (`basis.py:140-199`),
* BDM^k split into facet normal-moment functions (pseudo-inverse columns)
  and interior functions (SVD null space) (`basis.py:214-281`),
* the trace-free stress space with nt-trace in P^{k-1} (`basis.py:288-347`).

The interior BDM functions and the stress nt-bubbles are SVD null-space
vectors; they are only unique up to rotation, so the recipe (pinv + svd of
bitwise-identical constraint matrices) is kept identical to the reference.
`tests/test_fe_setup.py` pins the resulting coefficients against golden
vectors produced by the reference itself.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np
from scipy.special import eval_jacobi

from .quadrature import (REF_EDGE_LENGTHS, REF_EDGES, REF_NORMALS,
                         REF_TANGENTS, edge_points, edge_rule, triangle_rule)

# trace-free 2x2 generators: two symmetric deviatoric + one skew
DEV_COMPONENTS = np.array([[[1.0, 0.0], [0.0, -1.0]],
                           [[0.0, 1.0], [1.0, 0.0]],
                           [[0.0, 1.0], [-1.0, 0.0]]])


def shifted_legendre(nmax: int, t) -> np.ndarray:
    """L^2(0,1)-orthonormal Legendre polynomials L_0..L_nmax at t."""
    z = 2.0 * np.asarray(t, dtype=float) - 1.0
    P = np.empty((nmax + 1,) + z.shape)
    P[0] = 1.0
    if nmax >= 1:
        P[1] = z
    for n in range(1, nmax):
        P[n + 1] = ((2 * n + 1) * z * P[n] - n * P[n - 1]) / (n + 1)
    return P * np.sqrt(2.0 * np.arange(nmax + 1) + 1.0)[:, None]


def dubiner_pairs(k: int):
    return [(i, d - i) for d in range(k + 1) for i in range(d + 1)]


def _collapsed_legendre(imax, u, w, grad=False):
    """w^i P_i(u/w) by the homogeneous Legendre recurrence (and d/dx, d/dy
    with du = (2, 1), dw = (0, -1))."""
    A = np.empty((imax + 1,) + u.shape)
    A[0] = 1.0
    if imax >= 1:
        A[1] = u
    for i in range(2, imax + 1):
        A[i] = ((2 * i - 1) * u * A[i - 1] - (i - 1) * w * w * A[i - 2]) / i
    if not grad:
        return A, None
    du, dw = (2.0, 1.0), (0.0, -1.0)
    dA = np.zeros((imax + 1, 2) + u.shape)
    if imax >= 1:
        dA[1, 0], dA[1, 1] = du
    for i in range(2, imax + 1):
        for d in range(2):
            dA[i, d] = ((2 * i - 1) * (du[d] * A[i - 1] + u * dA[i - 1, d])
                        - (i - 1) * (2.0 * dw[d] * w * A[i - 2]
                                     + w * w * dA[i - 2, d])) / i
    return A, dA


def _dubiner_raw(k, pts, grad):
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    x, y = pts[:, 0], pts[:, 1]
    A, dA = _collapsed_legendre(k, 2.0 * x + y - 1.0, 1.0 - y, grad)
    z = 2.0 * y - 1.0
    pairs = dubiner_pairs(k)
    V = np.empty((len(pairs), len(x)))
    G = np.empty((len(pairs), len(x), 2)) if grad else None
    for m, (i, j) in enumerate(pairs):
        a = 2 * i + 1
        B = eval_jacobi(j, a, 0.0, z)
        V[m] = A[i] * B
        if grad:
            dB = (j + a + 1) * eval_jacobi(j - 1, a + 1, 1.0, z) if j else 0.0
            G[m, :, 0] = dA[i, 0] * B
            G[m, :, 1] = dA[i, 1] * B + A[i] * dB
    return V, G


@lru_cache(maxsize=None)
def _dubiner_norms(k: int) -> np.ndarray:
    rule = triangle_rule(2 * k + 2)
    V, _ = _dubiner_raw(k, rule.points, False)
    return np.sqrt(V * V @ rule.weights)


def dubiner_eval(k: int, pts, grad: bool = False):
    """Orthonormal Dubiner basis of degree k: values (M, n) [and (M, n, 2)]."""
    V, G = _dubiner_raw(k, pts, grad)
    nrm = _dubiner_norms(k)
    V /= nrm[:, None]
    if grad:
        G /= nrm[:, None, None]
        return V, G
    return V


def scalar_pk_eval(k: int, pts) -> np.ndarray:
    """Hierarchical scalar P^k (vertex, edge, bubble functions): (ndof, n)."""
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    x, y = pts[:, 0], pts[:, 1]
    lam = np.stack([1.0 - x - y, x, y])
    if k == 0:
        return np.ones((1, len(x)))
    rows = [lam[0], lam[1], lam[2]]
    for a, b in REF_EDGES:
        z = lam[b] - lam[a]
        for j in range(k - 1):
            rows.append(lam[a] * lam[b] * eval_jacobi(j, 1.0, 1.0, z))
    if k >= 3:
        bub = lam[0] * lam[1] * lam[2]
        for row in dubiner_eval(k - 3, pts):
            rows.append(bub * row)
    return np.array(rows)


class BdmBasis:
    """BDM^k: 3(k+1) facet functions with orthonormal normal-trace Legendre
    moments (pinv columns) followed by (k+1)(k-1) interior functions (SVD
    null space of the moment map)."""

    def __init__(self, k: int):
        self.degree = k
        M = (k + 1) * (k + 2) // 2
        self.nscalar, self.ndof = M, 2 * M
        self.n_edge, self.n_interior = k + 1, (k + 1) * (k - 1)
        er = edge_rule(2 * k + 2)
        leg = shifted_legendre(k, er.points)
        C = np.zeros((3 * (k + 1), 2 * M))
        for e in range(3):
            psi = dubiner_eval(k, edge_points(e, er.points))
            for q in range(k + 1):
                mom = psi @ (er.weights * leg[q] * REF_EDGE_LENGTHS[e])
                for c in range(2):
                    C[e * (k + 1) + q, c::2] = mom * REF_NORMALS[e][c]
        P = np.linalg.pinv(C)
        _, s, vt = np.linalg.svd(C)
        if int((s > s[0] * 1e-12).sum()) != 3 * (k + 1):
            raise RuntimeError("normal-moment matrix rank deficient")
        facet = P.T.reshape(3 * (k + 1), M, 2)
        interior = vt[3 * (k + 1):].reshape(-1, M, 2)
        self.coef = np.concatenate([facet, interior], axis=0)

    def eval(self, pts, grad=False):
        if grad:
            psi, dpsi = dubiner_eval(self.degree, pts, grad=True)
            return (np.einsum("fmd,mp->fpd", self.coef, psi),
                    np.einsum("fmd,mpe->fpde", self.coef, dpsi))
        return np.einsum("fmd,mp->fpd", self.coef, dubiner_eval(self.degree, pts))

    def div(self, pts):
        _, dpsi = dubiner_eval(self.degree, pts, grad=True)
        return np.einsum("fmd,mpd->fp", self.coef, dpsi)


class StressBasis:
    """Trace-free P^k stresses whose nt-trace is P^{k-1}: all of P^{k-1}
    times the 3 generators, plus the SVD null space of the degree-k nt
    Legendre moments."""

    def __init__(self, k: int):
        self.degree = k
        M = (k + 1) * (k + 2) // 2
        Mlow, ntop = k * (k + 1) // 2, k + 1
        self.nscalar = M
        er = edge_rule(2 * k + 2)
        legk = shifted_legendre(k, er.points)[k]
        R = np.zeros((3, 3 * ntop))
        for e in range(3):
            psi = dubiner_eval(k, edge_points(e, er.points))[Mlow:]
            mom = psi @ (er.weights * legk * REF_EDGE_LENGTHS[e])
            tDn = np.array([REF_TANGENTS[e] @ D @ REF_NORMALS[e]
                            for D in DEV_COMPONENTS])
            R[e] = np.outer(mom, tDn).ravel()
        _, s, vt = np.linalg.svd(R)
        if int((s > max(s[0], 1.0) * 1e-12).sum()) != 3:
            raise RuntimeError("nt-moment constraint matrix rank deficient")
        low = np.zeros((3 * Mlow, M, 3))
        low[np.arange(3 * Mlow), np.repeat(np.arange(Mlow), 3),
            np.tile(np.arange(3), Mlow)] = 1.0
        top = np.zeros((len(vt) - 3, M, 3))
        top[:, Mlow:, :] = vt[3:].reshape(-1, ntop, 3)
        self.coef = np.concatenate([low, top], axis=0)
        self.ndof = self.coef.shape[0]

    def components(self, pts) -> np.ndarray:
        """c[s, p, a]: coordinates of basis function s on the generators."""
        return np.einsum("fma,mp->fpa", self.coef, dubiner_eval(self.degree, pts))

    def eval(self, pts):
        return np.einsum("fpa,aij->fpij", self.components(pts), DEV_COMPONENTS)

    def div(self, pts):
        _, dpsi = dubiner_eval(self.degree, pts, grad=True)
        return np.einsum("fma,mpj,aij->fpi", self.coef, dpsi, DEV_COMPONENTS)


@lru_cache(maxsize=None)
def bdm_basis(k: int) -> BdmBasis:
    return BdmBasis(k)


@lru_cache(maxsize=None)
def sigma_basis(k: int) -> StressBasis:
    if k < 2:
        raise ValueError("stress basis needs degree >= 2")
    return StressBasis(k)
