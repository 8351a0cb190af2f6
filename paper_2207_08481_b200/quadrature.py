"""Reference-cell quadrature (host setup, not on the GPU hot path).

Restates the rules of the reference `quadrature.py` (Gauss-Legendre on the
unit interval, `quadrature.py:50-54`; collapsed Gauss x Gauss-Jacobi(1,0) on
the unit triangle, `quadrature.py:57-83`) so that the element tables built
from them agree with the reference to the last bits.  Point order on the
triangle is xi-major / eta-minor, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.special import roots_jacobi

SQRT_HALF = 1.0 / np.sqrt(2.0)

# reference triangle (0,0), (1,0), (0,1); local edge e is opposite vertex e
REF_VERTICES = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
REF_EDGES = ((1, 2), (2, 0), (0, 1))
REF_NORMALS = np.array([[SQRT_HALF, SQRT_HALF], [-1.0, 0.0], [0.0, -1.0]])
REF_TANGENTS = np.array([[-SQRT_HALF, SQRT_HALF], [0.0, -1.0], [1.0, 0.0]])
REF_EDGE_LENGTHS = np.array([np.sqrt(2.0), 1.0, 1.0])


@dataclass(frozen=True)
class EdgeRule:
    points: np.ndarray
    weights: np.ndarray
    exactness: int


@dataclass(frozen=True)
class TriangleRule:
    points: np.ndarray
    weights: np.ndarray
    exactness: int


def _npts(exactness: int) -> int:
    return exactness // 2 + 1


def edge_rule(exactness: int) -> EdgeRule:
    """Gauss-Legendre on [0, 1] with n = exactness//2 + 1 points."""
    n = _npts(exactness)
    x, w = np.polynomial.legendre.leggauss(n)
    return EdgeRule(points=0.5 * (x + 1.0), weights=0.5 * w,
                    exactness=2 * n - 1)


def triangle_rule(exactness: int) -> TriangleRule:
    """Duffy-collapsed product rule: xi Gauss-Legendre, eta Gauss-Jacobi
    with weight (1 - eta)."""
    n = _npts(exactness)
    gx, gw = np.polynomial.legendre.leggauss(n)
    xi, w_xi = 0.5 * (gx + 1.0), 0.5 * gw
    jx, jw = roots_jacobi(n, 1.0, 0.0)
    eta, w_eta = 0.5 * (jx + 1.0), 0.25 * jw
    XI, ETA = np.meshgrid(xi, eta, indexing="ij")
    WX, WE = np.meshgrid(w_xi, w_eta, indexing="ij")
    pts = np.stack([(XI * (1.0 - ETA)).ravel(), ETA.ravel()], axis=1)
    return TriangleRule(points=pts, weights=(WX * WE).ravel(),
                        exactness=2 * n - 1)


def edge_points(edge: int, s: np.ndarray) -> np.ndarray:
    """Reference-cell points of local edge `edge` at parameters s in [0,1]."""
    a, b = REF_EDGES[edge]
    va, vb = REF_VERTICES[a], REF_VERTICES[b]
    return va[None, :] + np.asarray(s, dtype=float)[:, None] * (vb - va)[None, :]
