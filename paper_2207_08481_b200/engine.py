"""Device-level operations over element batches (thin wrappers of the C ABI).

Layouts in HBM (all float64, element-major so one element is one contiguous
record that a single 1-D bulk async copy can move):

* element record  [msig ns*ns | bws nw*ns | bus nu*ns | bhs nh*ns | adiv nu*nu],
  each segment padded to an even length (`record_layout`);
* packed symmetric matrices: lower triangle, row-major, stride padded to an
  even length (S_T: `st_stride(k)`);
* geometry weights [nt][N_WEIGHTS] (`refblocks.element_weights`).
"""

from __future__ import annotations

import numpy as np

from . import _abi
from .refblocks import (N_WEIGHTS, W_ADIV, W_BHS, W_BUSE, W_BWS, W_MSIG,
                        W_ONE, BlockRefs, local_sizes)


def _even(n):
    return (n + 1) & ~1


def record_layout(k: int) -> dict:
    z = local_sizes(k)
    ns, nw, nu, nh = z["ns"], z["nw"], z["nu"], z["nh"]
    off, o = {}, 0
    for name, size in (("msig", ns * ns), ("bws", nw * ns), ("bus", nu * ns),
                       ("bhs", nh * ns), ("adiv", nu * nu)):
        off[name] = o
        o += _even(size)
    off["len"] = o
    return off


def st_stride(k: int) -> int:
    n = local_sizes(k)["nloc"]
    return _even(n * (n + 1) // 2)


def packed_stride(n: int) -> int:
    return _even(n * (n + 1) // 2)


def tril_index(n: int):
    """(rows, cols) of the lower-packed row-major order."""
    return np.tril_indices(n)


def pack_sym(M: np.ndarray, stride: int = None) -> np.ndarray:
    """(..., n, n) -> (..., stride) lower-packed."""
    n = M.shape[-1]
    r, c = np.tril_indices(n)
    P = M[..., r, c]
    stride = stride or packed_stride(n)
    if stride > P.shape[-1]:
        P = np.concatenate([P, np.zeros(P.shape[:-1] + (stride - P.shape[-1],))], -1)
    return P


def unpack_sym(P: np.ndarray, n: int) -> np.ndarray:
    r, c = np.tril_indices(n)
    M = np.zeros(P.shape[:-1] + (n, n))
    M[..., r, c] = P[..., :len(r)]
    M[..., c, r] = P[..., :len(r)]
    return M


def pack_records(k, msig, bws, bus, bhs, adiv) -> np.ndarray:
    """Host blocks (nt, ...) -> element records (nt, len)."""
    L = record_layout(k)
    nt = len(msig)
    R = np.zeros((nt, L["len"]))
    for name, blk in (("msig", msig), ("bws", bws), ("bus", bus), ("bhs", bhs),
                      ("adiv", adiv)):
        flat = np.asarray(blk, dtype=float).reshape(nt, -1)
        R[:, L[name]:L[name] + flat.shape[1]] = flat
    return R


def unpack_records(k, R):
    L = record_layout(k)
    z = local_sizes(k)
    ns, nw, nu, nh = z["ns"], z["nw"], z["nu"], z["nh"]
    nt = len(R)
    get = lambda name, shape: R[:, L[name]:L[name] + shape[0] * shape[1]].reshape(nt, *shape)
    return (get("msig", (ns, ns)), get("bws", (nw, ns)), get("bus", (nu, ns)),
            get("bhs", (nh, ns)), get("adiv", (nu, nu)))


def block_program(refs: BlockRefs, rel_drop: float = 1e-15):
    """CSR program (ptr, widx, coef) with one row per record entry:
    rec[q] = sum_p W[widx[p]] * coef[p].  Entries below rel_drop * max|ref|
    of their block (quadrature noise of structural zeros) are dropped."""
    k = refs.k
    L = record_layout(k)
    rows = [[] for _ in range(L["len"])]

    def add(off, ref, widx):
        ref = np.asarray(ref, dtype=float)
        tol = rel_drop * max(np.abs(ref).max(), 1e-300)
        flat = ref.reshape(ref.shape[0], -1) if ref.ndim > 1 else ref[None]
        for w, row in zip(widx, flat):
            nz = np.flatnonzero(np.abs(row) > tol)
            for q in nz:
                rows[off + q].append((w, row[q]))

    add(L["msig"], refs.msig, [W_MSIG + r for r in range(6)])
    add(L["bws"], refs.bws, [W_BWS + a for a in range(3)])
    add(L["bus"], refs.bus_vol[None], [W_ONE])
    add(L["bus"], refs.bus_edge.reshape(9, *refs.bus_vol.shape),
        [W_BUSE + r for r in range(9)])
    ns = refs.bhs.shape[-1]
    for e in range(3):
        # rows of edge e: bhs[e*k:(e+1)*k, :]
        for a in range(3):
            full = np.zeros((3 * k, ns))
            full[e * k:(e + 1) * k] = refs.bhs[e, a]
            add(L["bhs"], full[None], [W_BHS + 3 * e + a])
    add(L["adiv"], refs.adiv[None], [W_ADIV])
    ptr = np.zeros(L["len"] + 1, dtype=np.int32)
    ptr[1:] = np.cumsum([len(r) for r in rows])
    widx = np.array([w for r in rows for w, _ in r], dtype=np.int32)
    coef = np.array([v for r in rows for _, v in r], dtype=float)
    return ptr, widx, coef


# ------------------------------------------------------------- device calls


def _t():
    import torch
    return torch


def to_dev(a, dtype=None):
    torch = _t()
    a = np.ascontiguousarray(a)
    t = torch.from_numpy(a)
    if dtype is not None:
        t = t.to(dtype)
    return t.to("cuda", non_blocking=False)


def check_lib_layout(k: int):
    L = record_layout(k)
    if _abi.call("mcs_record_len", k) != L["len"] or \
            _abi.call("mcs_st_stride", k) != st_stride(k):
        raise _abi.McsError("record layout mismatch between Python and libmcsgpu")


def element_records(nt: int, W_dev, prog_dev, k: int, out=None, stream=None):
    torch = _t()
    L = record_layout(k)
    if out is None:
        out = torch.empty((nt, L["len"]), dtype=torch.float64, device="cuda")
    ptr, widx, coef = prog_dev
    _abi.call("mcs_element_blocks", nt, N_WEIGHTS, _abi.ptr(W_dev), L["len"],
              _abi.ptr(ptr), _abi.ptr(widx), _abi.ptr(coef), _abi.ptr(out),
              _abi.stream(stream))
    return out


def condense(k: int, records, out=None, info=None, stream=None):
    """S_T (packed, stride st_stride(k)) of every element record."""
    torch = _t()
    nt = records.shape[0]
    check_lib_layout(k)
    if out is None:
        out = torch.empty((nt, st_stride(k)), dtype=torch.float64, device="cuda")
    if info is None:
        info = torch.empty(nt, dtype=torch.int32, device="cuda")
    _abi.call("mcs_condense", k, nt, _abi.ptr(records), _abi.ptr(out),
              _abi.ptr(info), _abi.stream(stream))
    return out, info


def spd_schur(n: int, m: int, A_packed, B, out=None, info=None, stream=None):
    """S = B^T A^-1 B per element (A lower-packed, B n x m row-major)."""
    torch = _t()
    batch = A_packed.shape[0]
    if out is None:
        out = torch.empty((batch, m * (m + 1) // 2), dtype=torch.float64, device="cuda")
    if info is None:
        info = torch.empty(batch, dtype=torch.int32, device="cuda")
    _abi.call("mcs_spd_schur_batched", n, m, batch, _abi.ptr(A_packed), _abi.ptr(B),
              _abi.ptr(out), _abi.ptr(info), _abi.stream(stream))
    return out, info
