"""2D triangulations with canonically oriented facets (host setup).

Array-at-a-time restatement of the reference mesh module
(`mesh.py:106-176` `_build_mesh`, `mesh.py:185-208` `build_structured`,
`mesh.py:257-288` `classify_boundary`).  The numbering conventions are the
reference's, because every global dof index on the GPU derives from them:

* facets are numbered in order of first appearance when the triangles are
  walked in order with local edges (1,2), (2,0), (0,1);
* the facet normal points from the lower- to the higher-numbered incident
  triangle (outward on the boundary), the tangent is the normal rotated by
  +90 degrees, and the facet parameter starts at the endpoint from which the
  tangent points along the edge.

The loops of the reference are replaced by sorting / vectorised numpy so the
BASELINE meshes (up to 131k triangles) build in well under a second.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

LOCAL_EDGES = np.array([[1, 2], [2, 0], [0, 1]])


class MeshError(Exception):
    pass


@dataclass(frozen=True)
class Mesh:
    vertices: np.ndarray
    triangles: np.ndarray
    facets: np.ndarray
    facet_tri: np.ndarray
    facet_normal: np.ndarray = field(default=None, repr=False)
    facet_tangent: np.ndarray = field(default=None, repr=False)
    facet_length: np.ndarray = field(default=None, repr=False)
    facet_start: np.ndarray = field(default=None, repr=False)
    tri_facets: np.ndarray = field(default=None, repr=False)
    h_max: float = field(default=None)

    @property
    def num_vertices(self):
        return len(self.vertices)

    @property
    def num_triangles(self):
        return len(self.triangles)

    @property
    def num_facets(self):
        return len(self.facets)

    @property
    def boundary_facets(self):
        return np.flatnonzero(self.facet_tri[:, 1] < 0)

    @property
    def interior_facets(self):
        return np.flatnonzero(self.facet_tri[:, 1] >= 0)

    def facet_midpoints(self):
        return 0.5 * (self.vertices[self.facets[:, 0]]
                      + self.vertices[self.facets[:, 1]])

    def facet_end(self):
        """The endpoint that is not `facet_start`, per facet."""
        a = self.facet_start
        return np.where(self.facets[:, 0] != a, self.facets[:, 0],
                        self.facets[:, 1])

    def triangle_area(self):
        p = self.vertices[self.triangles]
        d1, d2 = p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]
        return 0.5 * (d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0])

    def triangle_diameter(self):
        p = self.vertices[self.triangles]
        e = np.stack([np.linalg.norm(p[:, 1] - p[:, 2], axis=1),
                      np.linalg.norm(p[:, 2] - p[:, 0], axis=1),
                      np.linalg.norm(p[:, 0] - p[:, 1], axis=1)])
        return e.max(axis=0)


def _build(vertices, triangles) -> Mesh:
    V = np.asarray(vertices, dtype=float)
    T = np.asarray(triangles, dtype=np.int64)
    nt = len(T)
    P = V[T]
    d1, d2 = P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]
    if np.any(0.5 * (d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0]) <= 0):
        raise MeshError("triangle with non-positive orientation")

    # all (triangle, local edge) pairs in walk order, keyed by sorted vertices
    ends = T[:, LOCAL_EDGES].reshape(-1, 2)
    lo, hi = ends.min(axis=1), ends.max(axis=1)
    key = lo * (len(V) + 1) + hi
    uniq, first, inv, counts = np.unique(key, return_index=True,
                                         return_inverse=True, return_counts=True)
    if np.any(counts > 2):
        raise MeshError("facet with more than two incident triangles")
    order = np.argsort(first, kind="stable")          # first-appearance order
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    fid = rank[inv]                                   # facet id per (t, le)
    nf = len(uniq)
    tri_facets = fid.reshape(nt, 3)

    facets = np.stack([lo, hi], axis=1)[first[order]]
    tri_of = np.repeat(np.arange(nt), 3)
    facet_tri = -np.ones((nf, 2), dtype=np.int64)
    walk = np.argsort(fid, kind="stable")             # per facet, walk order
    fs = fid[walk]
    is_first = np.r_[True, fs[1:] != fs[:-1]]
    facet_tri[fs[is_first], 0] = tri_of[walk[is_first]]
    facet_tri[fs[~is_first], 1] = tri_of[walk[~is_first]]

    if len(V) - nf + nt != 1:
        raise MeshError("Euler relation violated: domain not simply connected?")

    cen = P.mean(axis=1)
    va, vb = V[facets[:, 0]], V[facets[:, 1]]
    d = vb - va
    length = np.linalg.norm(d, axis=1)
    n = np.stack([d[:, 1], -d[:, 0]], axis=1) / length[:, None]
    t0, t1 = facet_tri[:, 0], facet_tri[:, 1]
    ref = np.where((t1 < 0)[:, None], 0.5 * (va + vb) - cen[t0],
                   cen[np.maximum(t1, 0)] - cen[t0])
    n = np.where((np.einsum("fi,fi->f", n, ref) < 0)[:, None], -n, n)
    tan = np.stack([-n[:, 1], n[:, 0]], axis=1)
    start = np.where(np.einsum("fi,fi->f", tan, d) > 0, facets[:, 0], facets[:, 1])

    edge_len = np.stack([np.linalg.norm(P[:, 1] - P[:, 0], axis=1),
                         np.linalg.norm(P[:, 2] - P[:, 1], axis=1),
                         np.linalg.norm(P[:, 0] - P[:, 2], axis=1)])
    return Mesh(vertices=V, triangles=T, facets=facets, facet_tri=facet_tri,
                facet_normal=n, facet_tangent=tan, facet_length=length,
                facet_start=start, tri_facets=tri_facets,
                h_max=float(edge_len.max()))


def from_arrays(vertices, triangles) -> Mesh:
    return _build(vertices, triangles)


def build_structured(nx: int, ny: int, rect=(0.0, 0.0, 1.0, 1.0)) -> Mesh:
    """Rectangle split into nx*ny cells, each cut along the lower-left to
    upper-right diagonal; vertex (i, j) has id i*(ny+1)+j."""
    if nx < 1 or ny < 1:
        raise ValueError("nx, ny must be >= 1")
    x0, y0, x1, y1 = rect
    if not (x1 > x0 and y1 > y0):
        raise ValueError("degenerate rectangle")
    xx, yy = np.meshgrid(np.linspace(x0, x1, nx + 1),
                         np.linspace(y0, y1, ny + 1), indexing="ij")
    I, J = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    v00 = (I * (ny + 1) + J).ravel()
    v10, v01 = v00 + (ny + 1), v00 + 1
    v11 = v10 + 1
    tris = np.empty((2 * nx * ny, 3), dtype=np.int64)
    tris[0::2] = np.stack([v00, v10, v11], axis=1)
    tris[1::2] = np.stack([v00, v11, v01], axis=1)
    return _build(np.stack([xx.ravel(), yy.ravel()], axis=1), tris)


def jittered_structured(n: int, amplitude: float, seed: int) -> Mesh:
    """BASELINE config 2 mesh: build_structured(n, n) with the interior
    vertices (x, y in (eps, 1-eps), vertex-id order) moved by
    uniform(-amplitude*h, amplitude*h) from default_rng(seed)."""
    base = build_structured(n, n)
    v = base.vertices.copy()
    eps, h = 1e-12, 1.0 / n
    inner = np.flatnonzero((v[:, 0] > eps) & (v[:, 0] < 1 - eps)
                           & (v[:, 1] > eps) & (v[:, 1] < 1 - eps))
    rng = np.random.default_rng(seed)
    v[inner] += rng.uniform(-amplitude * h, amplitude * h, size=(len(inner), 2))
    return from_arrays(v, base.triangles)


@dataclass(frozen=True)
class BoundaryRegions:
    dirichlet_facets: frozenset
    neumann_facets: frozenset
    tilde_neumann_facets: frozenset
    dirichlet_value: Optional[Callable] = None
    mean_zero_pressure: bool = False

    def kind(self, f: int) -> str:
        for name, s in (("D", self.dirichlet_facets), ("N", self.neumann_facets),
                        ("NT", self.tilde_neumann_facets)):
            if f in s:
                return name
        return "0"


def classify_boundary(mesh: Mesh, dirichlet=None, neumann=None,
                      tilde_neumann=None, dirichlet_value=None,
                      mean_zero_pressure=False,
                      allow_no_dirichlet=False) -> BoundaryRegions:
    """Partition boundary facets by midpoint predicates; each boundary facet
    must match exactly one (reference `mesh.py:257-288`)."""
    mids = mesh.facet_midpoints()
    named = [("D", dirichlet), ("N", neumann), ("NT", tilde_neumann)]
    out = {"D": set(), "N": set(), "NT": set()}
    for f in mesh.boundary_facets:
        hit = [nm for nm, pred in named if pred is not None and pred(mids[f])]
        if len(hit) != 1:
            raise MeshError("boundary facet %d at %s matched %d region predicates"
                            % (f, mids[f], len(hit)))
        out[hit[0]].add(int(f))
    if not out["D"] and not allow_no_dirichlet:
        raise MeshError("no Dirichlet boundary configured")
    if not (out["N"] or out["NT"] or mean_zero_pressure or allow_no_dirichlet):
        raise MeshError("pure Dirichlet problem needs mean_zero_pressure=True")
    return BoundaryRegions(frozenset(out["D"]), frozenset(out["N"]),
                           frozenset(out["NT"]), dirichlet_value,
                           mean_zero_pressure)
