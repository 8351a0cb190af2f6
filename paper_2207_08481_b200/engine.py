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


def srecord_layout(k: int) -> dict:
    """Compact record of the structured condensation (csrc/condense_struct.cu):
    [s (3) + pad | A_m 3x3 (ml blocks) | Mb (nb x nb) | Bsig = [bus; bhs] |
    adiv], every segment even.  ml = k(k+1)/2 low stress blocks, nb = 3k
    nt-bubbles, s = detJ skew(T_a) (the bws direction)."""
    z = local_sizes(k)
    ml, nb = k * (k + 1) // 2, 3 * k
    off, o = {}, 0
    for name, size in (("s", 4), ("A", 9 * ml), ("Mb", nb * nb),
                       ("B", z["nloc"] * z["ns"]), ("adiv", z["nu"] ** 2)):
        off[name] = o
        o += _even(size)
    off["len"] = o
    off["ml"], off["nb"] = ml, nb
    return off


def structure_error(msig, bws, k: int) -> float:
    """Relative size of the entries the structured condensation ignores:
    msig off its 3x3 / bubble diagonal blocks, bws outside the low columns,
    and bws row blocks not parallel to one 3-vector s (Phi (x) s).  ~1e-15 for
    element blocks of the reference spaces (basis.py:288-337)."""
    msig = np.asarray(msig, dtype=float)
    bws = np.asarray(bws, dtype=float)
    ml = k * (k + 1) // 2
    nl = 3 * ml
    mask = np.zeros(msig.shape[-2:], dtype=bool)
    for m in range(ml):
        mask[3 * m:3 * m + 3, 3 * m:3 * m + 3] = True
    mask[nl:, nl:] = True
    scale = np.abs(msig).max(axis=(-2, -1)) + 1e-300
    err = (np.abs(np.where(mask, 0.0, msig)).max(axis=(-2, -1)) / scale).max()
    bl = bws[..., :nl].reshape(bws.shape[:-1] + (ml, 3))
    bscale = np.abs(bws).max(axis=(-2, -1)) + 1e-300
    err = max(err, (np.abs(bws[..., nl:]).max(axis=(-2, -1)) / bscale).max()
              if bws.shape[-1] > nl else 0.0)
    s = _bws_direction(bws, k)
    proj = bl - np.einsum("...wmc,...c,...d->...wmd", bl, s, s)
    return float(max(err, (np.abs(proj).max(axis=(-3, -2, -1)) / bscale).max()))


def _bws_direction(bws, k):
    """Unit 3-vector s of bws = Phi (x) s, from its largest row block."""
    ml = k * (k + 1) // 2
    bl = np.asarray(bws)[..., :3 * ml].reshape(np.shape(bws)[:-1] + (ml, 3))
    flat = bl.reshape(bl.shape[:-3] + (-1, 3))
    j = np.argmax(np.linalg.norm(flat, axis=-1), axis=-1)
    s = np.take_along_axis(flat, j[..., None, None], axis=-2)[..., 0, :]
    return s / np.linalg.norm(s, axis=-1, keepdims=True)


def pack_srecords(k, msig, bws, bus, bhs, adiv) -> np.ndarray:
    """Host blocks (nt, ...) -> compact structured records (nt, len)."""
    L = srecord_layout(k)
    ml, nb = L["ml"], L["nb"]
    msig = np.asarray(msig, dtype=float)
    nt = len(msig)
    R = np.zeros((nt, L["len"]))
    R[:, 0:3] = _bws_direction(bws, k)
    nl = 3 * ml
    for m in range(ml):
        R[:, L["A"] + 9 * m:L["A"] + 9 * m + 9] = \
            msig[:, 3 * m:3 * m + 3, 3 * m:3 * m + 3].reshape(nt, 9)
    R[:, L["Mb"]:L["Mb"] + nb * nb] = msig[:, nl:, nl:].reshape(nt, -1)
    B = np.concatenate([np.asarray(bus, float), np.asarray(bhs, float)], axis=1)
    R[:, L["B"]:L["B"] + B[0].size] = B.reshape(nt, -1)
    a = np.asarray(adiv, float).reshape(nt, -1)
    R[:, L["adiv"]:L["adiv"] + a.shape[1]] = a
    return R


def fused_table_layout(k: int) -> dict:
    """Reference-cell tables of the fused warp-per-element kernel
    (csrc/condense_fused.cu FTab): G4 [NR][ns][4] = (base, T_0, T_1, T_2)
    per Bsig entry (rows >= nloc zero) | Adiv [nu][nu] | MbRef [6][nb][nb] |
    ARef [6][ml][9]."""
    z = local_sizes(k)
    ml, nb, ns, nu = k * (k + 1) // 2, 3 * k, z["ns"], z["nu"]
    NR = (z["nloc"] + 7) // 8 * 8
    off, o = {"NR": NR}, 0
    for name, size in (("G4", 4 * NR * ns), ("adiv", nu * nu),
                       ("Mb", 6 * nb * nb), ("A", 6 * 9 * ml)):
        off[name] = o
        o += _even(size)
    off["len"] = o
    return off


FUSED_ZERO_SLOT = 30          # weight slots 30..35 read as zero in the fused kernel


def fused_tables(refs: BlockRefs):
    """(tables float64 [len], row_woff int32 [NR]) for the fused kernel
    (row_woff documents the weight slots; the kernel derives them from k).

    Bsig row i = base[i] + sum_a W[row_woff[i] + a] * T_a[i]: the volume part
    of bus (J-invariant) plus the edge term -<s_nn, u_n> of the edge the
    facet dof i sits on (weights W_BUSE + 3e + a), or the bhs rows of edge e
    (weights W_BHS + 3e + a); interior rows read the zero slots."""
    k = refs.k
    z = local_sizes(k)
    L = fused_table_layout(k)
    NR, ns, nu, nloc, n_em = L["NR"], z["ns"], z["nu"], z["nloc"], z["n_em"]
    ml, nb = k * (k + 1) // 2, 3 * k
    nl = 3 * ml
    tab = np.zeros(L["len"])
    base = np.zeros((NR, ns))
    T = np.zeros((3, NR, ns))
    woff = np.full(NR, FUSED_ZERO_SLOT, dtype=np.int32)
    base[:nu] = refs.bus_vol
    scale = np.abs(refs.bus_edge).max()
    for e in range(3):
        rows = np.arange(e * (k + 1), (e + 1) * (k + 1))
        for a in range(3):
            E = refs.bus_edge[e, a]
            other = np.delete(E, rows, axis=0)
            if other.size and np.abs(other).max() > 1e-13 * scale:
                raise ValueError("bus edge term not confined to the edge's facet dofs")
            T[a, rows] = E[rows]
            T[a, nu + e * k:nu + (e + 1) * k] = refs.bhs[e, a]
        woff[rows] = W_BUSE + 3 * e
        woff[nu + e * k:nu + (e + 1) * k] = W_BHS + 3 * e
    assert n_em == 3 * (k + 1) and nloc == nu + 3 * k
    # low dof 3m + a' is Dubiner function m times generator a', so the edge
    # terms act on generator a only: T_a[i][3m + a'] = delta_aa' Ehat[i][m].
    # The fused kernel stores one Ehat per (row, m) and relies on it.
    Tl = T[:, :, :nl].reshape(3, NR, ml, 3)
    for a in range(3):
        for b in range(3):
            dev = np.abs(Tl[a, :, :, b] - (Tl[0, :, :, 0] if a == b else 0.0)).max()
            if dev > 1e-13 * max(scale, 1.0):
                raise ValueError("edge tables do not have the generator-diagonal structure")
    tab[L["G4"]:L["G4"] + 4 * NR * ns] = np.stack([base, T[0], T[1], T[2]], -1).ravel()
    tab[L["adiv"]:L["adiv"] + nu * nu] = refs.adiv.ravel()
    tab[L["Mb"]:L["Mb"] + 6 * nb * nb] = refs.msig[:, nl:, nl:].ravel()
    A = np.stack([refs.msig[:, 3 * m:3 * m + 3, 3 * m:3 * m + 3] for m in range(ml)], 1)
    tab[L["A"]:L["A"] + 6 * 9 * ml] = A.ravel()
    return tab, woff


FUSED_DEGREES = (2, 3, 4)


def recovery_tables(refs: BlockRefs) -> np.ndarray:
    """Tables of the stress-recovery kernel (csrc/recover.cu RTab): the fused
    tables followed by Phi^-T (nw x ml), where bws = [Phi (x) s | 0]."""
    k = refs.k
    ml = k * (k + 1) // 2
    Phi = refs.bws[0][:, 0:3 * ml:3]                  # (nw, ml)
    PhiT = np.linalg.inv(Phi).T
    tab = fused_tables(refs)[0]
    out = np.zeros(len(tab) + _even(ml * ml))
    out[:len(tab)] = tab
    out[len(tab):len(tab) + ml * ml] = PhiT.ravel()
    return out


def recover_stress(k: int, nt: int, W_dev, tables_dev, codes_dev, x_dev, sig=None, om=None,
                   info=None, stream=None):
    """(sigma, omega) per element from a full velocity vector (csrc/recover.cu)."""
    torch = _t()
    if _abi.call("mcs_recover_table_len", k) != tables_dev.numel():
        raise _abi.McsError("recovery table layout mismatch between Python and libmcsgpu")
    z = local_sizes(k)
    dev = W_dev.device
    if sig is None:
        sig = torch.empty(nt * z["ns"], dtype=torch.float64, device=dev)
    if om is None:
        om = torch.empty(nt * z["nw"], dtype=torch.float64, device=dev)
    if info is None:
        info = torch.empty(nt, dtype=torch.int32, device=dev)
    _abi.call("mcs_recover_stress", k, nt, _abi.ptr(W_dev), W_dev.shape[1], _abi.ptr(tables_dev),
              _abi.ptr(codes_dev), _abi.ptr(x_dev), _abi.ptr(sig), _abi.ptr(om), _abi.ptr(info),
              _abi.stream(stream))
    return sig, om, info


def condense_gen_ds(k: int, nt: int, W_dev, tables_dev, stream=None):
    """k = 5, 6: S_T from the geometry weights AND the double Schur outputs
    (ext = [X | S_oo^-1], Sd_T) in one kernel (csrc/condense_struct.cu
    condense_gen_kernel<..., DS = true> + csrc/ds_warp.cuh).  info bit 0:
    singular stress block, bit 1: S_oo not SPD."""
    torch = _t()
    if _abi.call("mcs_fused_table_len", k) != fused_table_layout(k)["len"]:
        raise _abi.McsError("fused table layout mismatch between Python and libmcsgpu")
    dev = W_dev.device
    ST = torch.empty((nt, st_stride(k)), dtype=torch.float64, device=dev)
    ext = torch.empty((nt, _abi.call("mcs_ext_stride", k)), dtype=torch.float64, device=dev)
    Sd = torch.empty((nt, _abi.call("mcs_sd_stride", k)), dtype=torch.float64, device=dev)
    info = torch.empty(nt, dtype=torch.int32, device=dev)
    _abi.call("mcs_condense_gen_ds", k, nt, _abi.ptr(W_dev), W_dev.shape[1], _abi.ptr(tables_dev),
              _abi.ptr(ST), _abi.ptr(ext), _abi.ptr(Sd), _abi.ptr(info), _abi.stream(stream))
    return ST, ext, Sd, info


def condense_gen(k: int, nt: int, W_dev, tables_dev, ST=None, info=None, stream=None):
    """S_T from the geometry weights for any k (csrc/condense_struct.cu
    condense_gen_kernel: Bsig regenerated from the fused tables, no record
    in HBM); used for k = 5, 6."""
    torch = _t()
    if _abi.call("mcs_fused_table_len", k) != fused_table_layout(k)["len"]:
        raise _abi.McsError("fused table layout mismatch between Python and libmcsgpu")
    dev = W_dev.device
    if ST is None:
        ST = torch.empty((nt, st_stride(k)), dtype=torch.float64, device=dev)
    if info is None:
        info = torch.empty(nt, dtype=torch.int32, device=dev)
    _abi.call("mcs_condense_gen", k, nt, _abi.ptr(W_dev), W_dev.shape[1], _abi.ptr(tables_dev),
              _abi.ptr(ST), _abi.ptr(info), _abi.stream(stream))
    return ST, info


def condense_fused(k: int, nt: int, W_dev, tables_dev, ST=None, ext=None, Sd=None,
                   info=None, stream=None):
    """Weights -> S_T, ext = [X | S_oo^-1], Sd_T in one warp-per-element
    kernel (csrc/condense_fused.cu).  info bit 0: singular stress block,
    bit 1: interior velocity block not SPD."""
    torch = _t()
    if _abi.call("mcs_fused_table_len", k) != fused_table_layout(k)["len"]:
        raise _abi.McsError("fused table layout mismatch between Python and libmcsgpu")
    dev = W_dev.device
    if ST is None:
        ST = torch.empty((nt, st_stride(k)), dtype=torch.float64, device=dev)
    if ext is None:
        ext = torch.empty((nt, _abi.call("mcs_ext_stride", k)), dtype=torch.float64, device=dev)
    if Sd is None:
        Sd = torch.empty((nt, _abi.call("mcs_sd_stride", k)), dtype=torch.float64, device=dev)
    if info is None:
        info = torch.empty(nt, dtype=torch.int32, device=dev)
    _abi.call("mcs_condense_fused", k, nt, _abi.ptr(W_dev), W_dev.shape[1], _abi.ptr(tables_dev),
              _abi.ptr(ST), _abi.ptr(ext), _abi.ptr(Sd), _abi.ptr(info),
              _abi.stream(stream))
    return ST, ext, Sd, info


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


def _program(nrows, entries):
    rows = [[] for _ in range(nrows)]
    for q, w, v in entries:
        rows[q].append((w, v))
    ptr = np.zeros(nrows + 1, dtype=np.int32)
    ptr[1:] = np.cumsum([len(r) for r in rows])
    widx = np.array([w for r in rows for w, _ in r], dtype=np.int32)
    coef = np.array([v for r in rows for _, v in r], dtype=float)
    return ptr, widx, coef


def sblock_program(refs: BlockRefs, rel_drop: float = 1e-15):
    """CSR program of the compact structured record (`srecord_layout`):
    rec[q] = sum_p W[widx[p]] * coef[p] over the geometry weights."""
    k = refs.k
    L = srecord_layout(k)
    ml, nb = L["ml"], L["nb"]
    nl = 3 * ml
    ent = []

    def add(off, ref, widx):
        ref = np.asarray(ref, dtype=float)
        flat = ref.reshape(ref.shape[0], -1)
        tol = rel_drop * max(np.abs(ref).max(), 1e-300)
        for w, row in zip(widx, flat):
            for q in np.flatnonzero(np.abs(row) > tol):
                ent.append((off + int(q), w, float(row[q])))

    for a in range(3):                                   # s = detJ skew(T_a)
        ent.append((L["s"] + a, W_BWS + a, 1.0))
    wm = [W_MSIG + r for r in range(6)]
    blocks = np.stack([refs.msig[:, 3 * m:3 * m + 3, 3 * m:3 * m + 3] for m in range(ml)], 1)
    add(L["A"], blocks.reshape(6, -1), wm)
    add(L["Mb"], refs.msig[:, nl:, nl:], wm)
    ns = refs.bus_vol.shape[1]
    nu = refs.bus_vol.shape[0]
    add(L["B"], refs.bus_vol[None], [W_ONE])
    add(L["B"], refs.bus_edge.reshape(9, nu, ns), [W_BUSE + r for r in range(9)])
    for e in range(3):
        for a in range(3):
            full = np.zeros((3 * k, ns))
            full[e * k:(e + 1) * k] = refs.bhs[e, a]
            add(L["B"] + nu * ns, full[None], [W_BHS + 3 * e + a])
    add(L["adiv"], refs.adiv[None], [W_ADIV])
    return _program(L["len"], ent)


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


def element_srecords(nt: int, W_dev, sprog_dev, k: int, out=None, stream=None):
    """Compact structured records on the GPU from the geometry weights."""
    torch = _t()
    L = srecord_layout(k)
    if out is None:
        out = torch.empty((nt, L["len"]), dtype=torch.float64, device="cuda")
    ptr, widx, coef = sprog_dev
    _abi.call("mcs_element_blocks", nt, N_WEIGHTS, _abi.ptr(W_dev), L["len"],
              _abi.ptr(ptr), _abi.ptr(widx), _abi.ptr(coef), _abi.ptr(out),
              _abi.stream(stream))
    return out


def condense_struct(k: int, srecords, out=None, info=None, stream=None):
    """S_T (packed, stride st_stride(k)) of every compact structured record
    (csrc/condense_struct.cu: S_T = adiv + Y Y^T)."""
    torch = _t()
    nt = srecords.shape[0]
    if _abi.call("mcs_srec_len", k) != srecord_layout(k)["len"]:
        raise _abi.McsError("structured record layout mismatch between Python and libmcsgpu")
    if out is None:
        out = torch.empty((nt, st_stride(k)), dtype=torch.float64, device="cuda")
    if info is None:
        info = torch.empty(nt, dtype=torch.int32, device="cuda")
    _abi.call("mcs_condense_struct", k, nt, _abi.ptr(srecords), _abi.ptr(out),
              _abi.ptr(info), _abi.stream(stream))
    return out, info


def condense(k: int, records, out=None, info=None, stream=None):
    """S_T (packed, stride st_stride(k)) of every element record (general
    dense signed-Cholesky path, any SPD msig: csrc/condense.cu)."""
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
