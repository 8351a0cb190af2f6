"""Exact P1 coarse solve on the GPU.

The reference factorises the free P1 strain matrix with SuperLU and calls
`lu.solve` twice per preconditioner application (`preconditioners.py:111-118,
165-171`).  The coarse correction must stay exact for PCG iteration-count
parity, so this module builds a *multifrontal Cholesky factorisation* on the
host once per mesh and runs both triangular solves on the GPU:

* ordering: nested dissection by recursive coordinate bisection of the P1
  vertices (a general 2D-mesh ordering; separators are the vertices of one
  half adjacent to the other half);
* numeric: dense fronts per separator-tree node, L_SS = chol(F_SS),
  W = F_BS L_SS^-T, update U = F_BB - W W^T extend-added into the parent;
* storage for the solve: per node the explicit triangular inverse
  Linv = L_SS^-1 and W (and their transposes), so every solve step is a
  dense, coalesced GEMV (warp per row) instead of a latency-bound triangular
  recurrence;
* GPU schedule: one kernel per tree level and direction, one CTA per node:
  forward y_S = Linv (b_S - child updates), out_B = W y_S + pass-through;
  backward s = y_S - W^T x_B, x_S = Linv^T s.  Child contributions are
  gathered in a fixed order, so the solve is deterministic.

Small problems (n <= DENSE_MAX) use an explicit dense inverse instead.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import os

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import _abi, engine

DENSE_MAX = 1024
LEAF = int(os.environ.get("MCS_LEAF", "64"))   # max dofs of a nested-dissection leaf (A/B in PCG: 64 > 80 > 96)
TOP_MAX = int(os.environ.get("MCS_TOP_MAX", "4096"))   # dense-inverse top (A/B in PCG: 4096 > 2048)
# supernode amalgamation of the separator tree: "lo-hi[,lo-hi...]" merges, into
# every node of height hi, its descendants of height >= lo (one front, one
# level kernel instead of hi - lo + 1).  "" = none.
AMALG = os.environ.get("MCS_AMALG", "")


@dataclass
class _Node:
    own: np.ndarray                  # original dof ids eliminated here
    children: List["_Node"] = field(default_factory=list)
    s0: int = 0                      # first elimination position
    B: np.ndarray = None             # boundary (elimination positions, sorted)
    level: int = 0


def _nested_dissection(A: sp.csr_matrix, xy: np.ndarray, leaf: int) -> _Node:
    n = A.shape[0]

    def rec(dofs):
        if len(dofs) <= leaf:
            return _Node(own=np.sort(dofs))
        pts = xy[dofs]
        axis = int(np.argmax(pts.max(0) - pts.min(0)))
        order = np.lexsort((dofs, pts[:, axis]))
        half = len(dofs) // 2
        # keep the two components of a vertex on the same side
        cut = pts[order[half], axis]
        left_mask = pts[:, axis] < cut
        if left_mask.all() or not left_mask.any():
            left_mask = np.zeros(len(dofs), dtype=bool)
            left_mask[order[:half]] = True
        left, right = dofs[left_mask], dofs[~left_mask]
        if len(left) and len(right):
            sep_mask = np.asarray((A[left][:, right] != 0).sum(axis=1)).ravel() > 0
        else:
            sep_mask = np.zeros(len(left), dtype=bool)
        sep, left = left[sep_mask], left[~sep_mask]
        kids = [rec(part) for part in (left, right) if len(part)]
        return _Node(own=np.sort(sep), children=kids)

    return rec(np.arange(n))


def _heights(root):
    h = {}

    def walk(nd):
        h[id(nd)] = 1 + max([walk(c) for c in nd.children], default=-1)
        return h[id(nd)]

    walk(root)
    return h


def _amalgamate(root: _Node, spec: str) -> _Node:
    """Merge bands of the separator tree into supernodes (see AMALG): the
    merged node eliminates the union of the own dofs (descendants first), its
    children are the subtrees hanging below the band.  Any such merge keeps
    the factorisation exact (the front is dense); it trades a few more factor
    bytes for fewer dependent level kernels."""
    bands = []
    for part in filter(None, (q.strip() for q in spec.split(","))):
        lo, hi = (int(v) for v in part.split("-"))
        if not 0 <= lo < hi:
            raise ValueError(f"MCS_AMALG band {part!r}")
        bands.append((lo, hi))
    for lo, hi in sorted(bands, reverse=True):          # top bands first: heights below stay valid
        h = _heights(root)

        def absorb(nd, lo=lo, h=h):
            """own dofs (postorder) and hanging subtrees of nd's descendants of height >= lo"""
            own, kids = [], []
            for c in nd.children:
                if h[id(c)] >= lo:
                    o, k = absorb(c)
                    own += o + [c.own]
                    kids += k
                else:
                    kids.append(c)
            return own, kids

        def walk(nd, lo=lo, hi=hi, h=h):
            if h[id(nd)] == hi:
                own, kids = absorb(nd)
                nd.own = np.concatenate(own + [nd.own]) if own else nd.own
                nd.children = kids
            for c in nd.children:
                walk(c)

        walk(root)
    return root


def _postorder(root):
    out = []

    def walk(nd):
        for c in nd.children:
            walk(c)
        out.append(nd)

    walk(root)
    return out


@dataclass
class MultifrontalFactor:
    n: int
    perm: np.ndarray                 # elimination position -> original dof
    nodes: list
    levels: list                     # node indices per height
    A: object = None                 # the matrix (original dof order)
    dev: dict = None


def multifrontal_factor(A: sp.csr_matrix, xy: np.ndarray, leaf: int = LEAF) -> MultifrontalFactor:
    A = A.tocsr()
    n = A.shape[0]
    root = _nested_dissection(A, xy, leaf)
    if AMALG:
        root = _amalgamate(root, AMALG)
    nodes = _postorder(root)
    perm = np.concatenate([nd.own for nd in nodes]).astype(np.int64)
    pos = np.empty(n, dtype=np.int64)
    pos[perm] = np.arange(n)
    s = 0
    for nd in nodes:
        nd.s0 = s
        s += len(nd.own)
    Ap = A[perm][:, perm].tocsr()                # elimination order
    idx = {id(nd): i for i, nd in enumerate(nodes)}
    heights = [0] * len(nodes)
    updates = {}
    for i, nd in enumerate(nodes):
        ns = len(nd.own)
        S = np.arange(nd.s0, nd.s0 + ns)
        # structural boundary: later positions adjacent to S or in children's B
        cand = [Ap.indices[Ap.indptr[nd.s0]:Ap.indptr[nd.s0 + ns]]]
        cand += [c.B for c in nd.children]
        Bset = np.unique(np.concatenate(cand)) if cand else np.zeros(0, np.int64)
        B = Bset[Bset >= nd.s0 + ns]
        nd.B = B
        heights[i] = 1 + max([heights[idx[id(c)]] for c in nd.children], default=-1)
        nd.level = heights[i]
        nb = len(B)
        F = np.zeros((ns + nb, ns + nb))
        loc = np.full(n, -1, dtype=np.int64)
        loc[S] = np.arange(ns)
        loc[B] = ns + np.arange(nb)
        blk = Ap[nd.s0:nd.s0 + ns].tocoo()
        rows, cols = blk.row, loc[blk.col]
        keep = cols >= 0
        F[rows[keep], cols[keep]] += blk.data[keep]
        # symmetric part: (B, S) entries
        bmask = cols[keep] >= ns
        F[cols[keep][bmask], rows[keep][bmask]] += blk.data[keep][bmask]
        for c in nd.children:
            U = updates.pop(id(c))
            li = loc[c.B]
            F[np.ix_(li, li)] += U
        L = sla.cholesky(F[:ns, :ns], lower=True, check_finite=False) if ns else np.zeros((0, 0))
        W = sla.solve_triangular(L, F[ns:, :ns].T, lower=True, check_finite=False).T if ns else \
            np.zeros((nb, 0))
        if nb:
            updates[id(nd)] = F[ns:, ns:] - W @ W.T
        nd.Linv = sla.solve_triangular(L, np.eye(ns), lower=True, check_finite=False) if ns else L
        nd.L = L
        nd.W = W
    H = max(heights) + 1
    levels = [[i for i, h in enumerate(heights) if h == lv] for lv in range(H)]
    return MultifrontalFactor(n=n, perm=perm, nodes=nodes, levels=levels, A=A)


def _upload_multifrontal(F: MultifrontalFactor):
    """Flatten the factor into device arrays + per-level node lists.

    Per node: Linv packed lower (row-major), Linv^T packed upper (row-major),
    W (nb x ns) and W^T (ns x nb); gather sources: for every own position
    and every boundary row, the (<= 2) child update entries that land there.
    """
    nodes = F.nodes
    if max(len(nd.own) for nd in nodes) > 2048:
        raise ValueError("separator larger than the kernel's 2048-dof shared buffer")
    idx = {id(nd): i for i, nd in enumerate(nodes)}
    mats, off = [], 0
    out_off, oo = [], 0
    bo = 0
    node_tab = np.zeros((len(nodes), 10), dtype=np.int64)
    Bcat = []
    for i, nd in enumerate(nodes):
        ns, nb = len(nd.own), len(nd.B)
        r, c = np.tril_indices(ns)
        lo = nd.Linv[r, c]                                  # packed lower, row-major
        ru, cu = np.triu_indices(ns)
        up = nd.Linv.T[ru, cu]                              # packed upper, row-major
        # forward block [Linv | W] and backward block [W^T | Linv^T], each
        # starting on an even offset (16-byte aligned for the bulk copies of
        # coarse.cu mf_forward_s / mf_backward_s) and padded to even length
        pad = (len(lo) + nb * ns) % 2
        o_L = off; mats.append(lo); off += len(lo)
        o_W = off; mats.append(nd.W.ravel()); off += nb * ns
        mats.append(np.zeros(pad)); off += pad
        o_WT = off; mats.append(np.ascontiguousarray(nd.W.T).ravel()); off += nb * ns
        o_LT = off; mats.append(up); off += len(up)
        mats.append(np.zeros(pad)); off += pad
        node_tab[i] = [nd.s0, ns, nb, o_L, o_LT, o_W, o_WT, oo, bo, 0]
        out_off.append(oo)
        oo += nb
        bo += nb
        Bcat.append(nd.B)
    # gather sources per entry: one slot per child (2 in a plain separator
    # tree, more under amalgamated supernodes); the kernels read the count
    # from the node record
    nslot = max(2, max(len(nd.children) for nd in nodes))
    node_tab[:, 9] = nslot
    src_t = -np.ones((F.n, nslot), dtype=np.int64)
    src_o = -np.ones((max(oo, 1), nslot), dtype=np.int64)
    for i, nd in enumerate(nodes):
        ns = len(nd.own)
        loc = {int(p): r for r, p in enumerate(nd.B)}
        for slot, c in enumerate(nd.children):
            ci = idx[id(c)]
            for e, p in enumerate(c.B):
                p = int(p)
                src = out_off[ci] + e
                if nd.s0 <= p < nd.s0 + ns:
                    src_t[p, slot] = src
                else:
                    src_o[out_off[i] + loc[p], slot] = src
    torch = __import__("torch")
    H, top = _top_split(F)
    top_dev = None
    if top is not None:
        T, ptr, src, Sinv = top
        top_dev = dict(t=len(T), T=engine.to_dev(T.astype(np.int32)),
                       ptr=engine.to_dev(ptr.astype(np.int32)),
                       src=engine.to_dev(src.astype(np.int32) if len(src) else np.zeros(1, np.int32)),
                       Sinv=engine.to_dev(_pad_cols(Sinv, _abi.call("mcs_mf_top_ld", len(T)))),
                       g=torch.zeros(_abi.call("mcs_mf_top_ld", len(T)), dtype=torch.float64,
                                     device="cuda"))
    F.dev = dict(
        top=top_dev, H=H,
        mats=engine.to_dev(np.concatenate(mats) if mats else np.zeros(1)),
        nodes=engine.to_dev(node_tab),
        B=engine.to_dev(np.concatenate(Bcat).astype(np.int32) if oo else np.zeros(1, np.int32)),
        src_t=engine.to_dev(src_t.astype(np.int32)),
        src_o=engine.to_dev(src_o.astype(np.int32)),
        perm=engine.to_dev(F.perm.astype(np.int32)),
        levels=[(engine.to_dev(np.array(lv, dtype=np.int32)), len(lv),
                 max(len(nodes[i].own) for i in lv), max(len(nodes[i].B) for i in lv))
                for lv in F.levels[:H]],
        y=torch.empty(F.n, dtype=torch.float64, device="cuda"),
        xp=torch.empty(F.n, dtype=torch.float64, device="cuda"),
        out=torch.empty(max(oo, 1), dtype=torch.float64, device="cuda"),
        bytes=8 * off,
    )
    return F


def _pad_cols(S: np.ndarray, ld: int) -> np.ndarray:
    """Rows of S padded with zeros to ld columns (coarse.cu mf_top_solve)."""
    P = np.zeros((S.shape[0], ld))
    P[:, :S.shape[1]] = S
    return P


def _top_split(F: MultifrontalFactor, top_max: int = None):
    """Cut the separator tree at height H: nodes at height >= H (their own
    dofs T, at most top_max) are solved with the dense inverse of their
    Schur complement, which equals the T x T block of A^-1.  Returns H and
    (T positions, CSR gather sources of the frontier updates, Sinv)."""
    top_max = TOP_MAX if top_max is None else top_max
    nodes, levels = F.nodes, F.levels
    H = len(levels)
    size = 0
    while H > 0 and size + sum(len(nodes[i].own) for i in levels[H - 1]) <= top_max:
        H -= 1
        size += sum(len(nodes[i].own) for i in levels[H])
    if H == len(levels):
        raise ValueError("top separator larger than TOP_MAX")
    top_ids = [i for lv in levels[H:] for i in lv]
    T = np.sort(np.concatenate([np.arange(nodes[i].s0, nodes[i].s0 + len(nodes[i].own))
                                for i in top_ids]))
    tpos = -np.ones(F.n, dtype=np.int64)
    tpos[T] = np.arange(len(T))
    idx = {id(nd): i for i, nd in enumerate(nodes)}
    out_off, oo = [], 0
    for nd in nodes:
        out_off.append(oo)
        oo += len(nd.B)
    top_set = set(top_ids)
    lists = [[] for _ in range(len(T))]
    for i in top_ids:
        for c in nodes[i].children:
            ci = idx[id(c)]
            if ci in top_set:
                continue
            for e, p in enumerate(c.B):          # frontier node: B_c is inside T
                lists[tpos[int(p)]].append(out_off[ci] + e)
    ptr = np.zeros(len(T) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(l) for l in lists])
    src = np.array([s_ for l in lists for s_ in l], dtype=np.int64)
    # The top nodes' blocks form the Cholesky factor of the top Schur
    # complement S_T in the elimination order of T: L_T[S, S] = L_SS and
    # L_T[B, S] = W.  Then (A^-1)_TT = S_T^-1 = L_T^-T L_T^-1 (dense, t^3/3).
    Lt = np.zeros((len(T), len(T)))
    for i in top_ids:
        nd = nodes[i]
        S = tpos[np.arange(nd.s0, nd.s0 + len(nd.own))]
        Lt[np.ix_(S, S)] = nd.L
        if len(nd.B):
            Lt[np.ix_(tpos[nd.B], S)] = nd.W
    Li = sla.solve_triangular(Lt, np.eye(len(T)), lower=True, check_finite=False)
    Sinv = Li.T @ Li
    Sinv = 0.5 * (Sinv + Sinv.T)
    return H, (T, ptr, src, np.ascontiguousarray(Sinv))


class CoarseSolver:
    """`CoarseSolver` of the reference (`preconditioners.py:111-118`): holds
    the free coarse matrix and an exact GPU factorisation; `solve` accepts
    NumPy (compatibility) and `solve_dev` works on device vectors."""

    def __init__(self, matrix, kind, data, scale=1.0):
        self.matrix, self.kind, self.data, self.scale = matrix, kind, data, scale
        self.n = matrix.shape[0]

    def solve_dev(self, b, x, stream=None):
        st = _abi.stream(stream)
        if self.kind == "dense":
            _abi.call("mcs_dense_gemv", self.n, _abi.ptr(self.data), _abi.ptr(b), _abi.ptr(x), st)
        else:
            d = self.data.dev
            for ln, cnt, mns, mnb in d["levels"]:          # bottom levels, forward
                _abi.call("mcs_mf_forward", cnt, _abi.ptr(ln), _abi.ptr(d["nodes"]),
                          _abi.ptr(d["mats"]), _abi.ptr(d["src_t"]), _abi.ptr(d["src_o"]),
                          _abi.ptr(d["perm"]), _abi.ptr(b), _abi.ptr(d["y"]), _abi.ptr(d["out"]),
                          mns, mnb, st)
            tp = d["top"]                                  # dense top Schur complement
            _abi.call("mcs_mf_top", tp["t"], _abi.ptr(tp["T"]), _abi.ptr(d["perm"]), _abi.ptr(b),
                      _abi.ptr(tp["ptr"]), _abi.ptr(tp["src"]), _abi.ptr(d["out"]),
                      _abi.ptr(tp["g"]), _abi.ptr(tp["Sinv"]), _abi.ptr(d["xp"]), _abi.ptr(x), st)
            for ln, cnt, mns, mnb in reversed(d["levels"]):  # bottom levels, backward
                _abi.call("mcs_mf_backward", cnt, _abi.ptr(ln), _abi.ptr(d["nodes"]),
                          _abi.ptr(d["mats"]), _abi.ptr(d["B"]), _abi.ptr(d["perm"]),
                          _abi.ptr(d["y"]), _abi.ptr(d["xp"]), _abi.ptr(x), mns, mnb, st)
        if self.scale != 1.0:
            from .operators import axpby
            axpby(1.0 / self.scale, x, 0.0, x, stream)
        return x

    def solve(self, r):
        import torch
        b = torch.from_numpy(np.ascontiguousarray(r, dtype=np.float64)).cuda()
        x = torch.empty_like(b)
        return self.solve_dev(b, x).cpu().numpy()


def graph_coordinates(A: sp.csr_matrix) -> np.ndarray:
    """Stand-in vertex coordinates for the nested dissection when the caller
    has only the matrix (a reference `CoarseSolver`): BFS distances from two
    pseudo-peripheral vertices of the matrix graph.  Any bisection keeps the
    factorisation exact; this one keeps the separators small on mesh graphs."""
    from scipy.sparse.csgraph import breadth_first_order, shortest_path
    n = A.shape[0]
    G = (abs(A) + abs(A.T)).tocsr()
    order = breadth_first_order(G, 0, directed=False, return_predecessors=False)
    a = int(order[-1])
    da = shortest_path(G, unweighted=True, indices=a, directed=False)
    b = int(np.argmax(np.where(np.isfinite(da), da, -1)))
    db = shortest_path(G, unweighted=True, indices=b, directed=False)
    xy = np.stack([da, db], axis=1)
    xy[~np.isfinite(xy)] = 0.0
    return xy + 1e-3 * np.arange(n)[:, None] / max(n, 1)


def factorize_coarse(A: sp.csr_matrix, xy: np.ndarray, scale=1.0, kind=None,
                     leaf=LEAF) -> CoarseSolver:
    """Exact GPU factorisation of the free coarse matrix; `xy` = per-dof
    coordinates for the nested dissection (None: graph_coordinates(A))."""
    n = A.shape[0]
    kind = kind or ("dense" if n <= DENSE_MAX else "multifrontal")
    if kind == "dense":
        Ainv = np.linalg.inv(A.toarray())
        Ainv = 0.5 * (Ainv + Ainv.T)
        return CoarseSolver(A, "dense", engine.to_dev(Ainv), scale)
    if xy is None:
        xy = graph_coordinates(A)
    F = multifrontal_factor(A, xy, leaf=leaf)
    return CoarseSolver(A, "multifrontal", _upload_multifrontal(F), scale)
