"""Host emulation of the GPU multifrontal solve schedule (test helper only):
same level order, same child->parent gather rule, NumPy GEMVs."""
import numpy as np


def emulate_solve(F, b):
    nodes = F.nodes
    idx = {id(nd): i for i, nd in enumerate(nodes)}
    out_off, oo = [], 0
    for nd in nodes:
        out_off.append(oo)
        oo += len(nd.B)
    y, out, xp = np.zeros(F.n), np.zeros(max(oo, 1)), np.zeros(F.n)
    for lv in F.levels:
        for i in lv:
            nd = nodes[i]
            ns = len(nd.own)
            t = b[F.perm[nd.s0:nd.s0 + ns]].copy()
            loc = {int(p): r for r, p in enumerate(nd.B)}
            o_pass = np.zeros(len(nd.B))
            for c in nd.children:
                ci = idx[id(c)]
                for e, p in enumerate(c.B):
                    if nd.s0 <= p < nd.s0 + ns:
                        t[p - nd.s0] -= out[out_off[ci] + e]
                    else:
                        o_pass[loc[int(p)]] += out[out_off[ci] + e]
            y[nd.s0:nd.s0 + ns] = nd.Linv @ t
            out[out_off[i]:out_off[i] + len(nd.B)] = nd.W @ y[nd.s0:nd.s0 + ns] + o_pass
    for lv in reversed(F.levels):
        for i in lv:
            nd = nodes[i]
            ns = len(nd.own)
            s = y[nd.s0:nd.s0 + ns] - nd.W.T @ xp[nd.B]
            xp[nd.s0:nd.s0 + ns] = nd.Linv.T @ s
    x = np.zeros(F.n)
    x[F.perm] = xp
    return x


def emulate_hybrid(F, b):
    """The GPU schedule with the dense top: bottom forward, gather + dense
    inverse on the top dofs, bottom backward."""
    from paper_2207_08481_b200.coarse import _top_split
    H, (T, ptr, src, Sinv) = _top_split(F)
    nodes = F.nodes
    idx = {id(nd): i for i, nd in enumerate(nodes)}
    out_off, oo = [], 0
    for nd in nodes:
        out_off.append(oo)
        oo += len(nd.B)
    y, out, xp = np.zeros(F.n), np.zeros(max(oo, 1)), np.zeros(F.n)
    for lv in F.levels[:H]:
        for i in lv:
            nd = nodes[i]
            ns = len(nd.own)
            t = b[F.perm[nd.s0:nd.s0 + ns]].copy()
            loc = {int(p): r for r, p in enumerate(nd.B)}
            o_pass = np.zeros(len(nd.B))
            for c in nd.children:
                ci = idx[id(c)]
                for e, p in enumerate(c.B):
                    if nd.s0 <= p < nd.s0 + ns:
                        t[p - nd.s0] -= out[out_off[ci] + e]
                    else:
                        o_pass[loc[int(p)]] += out[out_off[ci] + e]
            y[nd.s0:nd.s0 + ns] = nd.Linv @ t
            out[out_off[i]:out_off[i] + len(nd.B)] = nd.W @ y[nd.s0:nd.s0 + ns] + o_pass
    g = b[F.perm[T]] - np.array([out[src[ptr[q]:ptr[q + 1]]].sum() for q in range(len(T))])
    xp[T] = Sinv @ g
    for lv in reversed(F.levels[:H]):
        for i in lv:
            nd = nodes[i]
            ns = len(nd.own)
            s = y[nd.s0:nd.s0 + ns] - nd.W.T @ xp[nd.B]
            xp[nd.s0:nd.s0 + ns] = nd.Linv.T @ s
    x = np.zeros(F.n)
    x[F.perm] = xp
    return x
