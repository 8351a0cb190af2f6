"""Drop-in `condense_sigma_omega` / `double_schur` / `CondensedSystem` on B200.

Reference: `condensation.py:26-239`.  Same entry points, same argument
meaning, same exceptions; the per-element work runs in the CUDA kernels of
`csrc/condense.cu` (A1 block generation + A3 elimination) and
`csrc/double_schur.cu` (A4), and the results stay resident in HBM:

  S_T    (nt, st_stride)  packed lower S_T per element
  ext    (nt, ext_stride) [X | S_oo^-1] per element
  Sd_T   (nt, sd_stride)  packed lower Sd_T per element

The assembled host CSR matrices the reference exposes (`S`, `Sd`, `B`) and the
per-element host lists (`ext`, `soo_dense`, `soo_chol`) are materialised
lazily from the device data only when a caller touches them (tests,
exports); the solver path never does.
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import scipy.sparse as sp

from . import _abi, engine
from .maps import element_maps, local_splits
from .refblocks import build_refs, element_weights, load_vectors, local_sizes


def _torch():
    import torch
    return torch


def _assemble(n, l2g, sg, mats):
    nt, m = l2g.shape
    vals = mats * sg[:, :, None] * sg[:, None, :]
    I = np.repeat(l2g, m, axis=1).ravel()
    J = np.tile(l2g, (1, m)).ravel()
    return sp.coo_matrix((vals.ravel(), (I, J)), shape=(n, n)).tocsr()


class CondensedSystem:
    """GPU-resident condensed system with the reference's attribute surface."""

    def __init__(self, fes, nu, S_dev, load, maps, refs, records=None):
        self.fes, self.nu = fes, nu
        z = local_sizes(fes.k)
        self.k, self.z = fes.k, z
        self.S_dev = S_dev                  # (nt, st_stride) float64 cuda
        self.records = records
        self.load = load
        self.maps = maps
        self.refs = refs
        self.vv_l2g, self.vv_signs = maps.vv_l2g, maps.vv_signs
        self.n_cpl_loc = z["ncpl"]
        self.nloc_u = z["nu"]
        self.ext_dev = None
        self.Sd_dev = None
        self.cpl_of_vv = None
        self.vv_of_cpl = None
        self._S = self._Sd = self._B = None
        self._dev_maps = None
        # double Schur outputs produced together with S_T by the fused
        # kernel (k <= 4); double_schur() publishes them
        self._pending_ds = None

    # -------------------------------------------------------------- indexing
    @property
    def n_vv(self):
        return self.fes.n_vv

    def free_mask_vv(self):
        return self.fes.vv_free

    def free_mask_cpl(self):
        return self.fes.vv_free[self.vv_of_cpl]

    def local_vv(self, x_full, t):
        return x_full[self.vv_l2g[t]] * self.vv_signs[t]

    def _local_splits(self):
        return local_splits(self.k)

    def dev_maps(self):
        """int32 device maps used by the operators (built once)."""
        if self._dev_maps is None:
            m = self.maps
            self._dev_maps = dict(
                vv_codes=engine.to_dev(m.vv_codes),
                bubble_idx=engine.to_dev(m.bubble_idx),
                cpl_codes=engine.to_dev(m.cpl_codes),
                c2v=engine.to_dev(m.cplfree_to_vvfree))
        return self._dev_maps

    # ------------------------------------------------- lazy host compatibility
    def S_T_host(self):
        return engine.unpack_sym(self.S_dev.cpu().numpy(), self.z["nloc"])

    @property
    def S(self):
        if self._S is None:
            self._S = _assemble(self.fes.n_vv, self.vv_l2g, self.vv_signs, self.S_T_host())
        return self._S

    @property
    def B(self):
        if self._B is None:
            fes = self.fes
            nt, nu_l = fes.mesh.num_triangles, self.z["nu"]
            bpu = self.refs.bpu
            vals = bpu[None] * self.vv_signs[:, None, :nu_l]
            rows = np.repeat(fes.dof_q.loc2glob, nu_l, axis=1).ravel()
            cols = np.tile(self.vv_l2g[:, :nu_l], (1, bpu.shape[0])).ravel()
            self._B = sp.coo_matrix((vals.ravel(), (rows, cols)),
                                    shape=(fes.dof_q.ndof, fes.n_vv)).tocsr()
        return self._B

    @property
    def Sd(self):
        if self.Sd_dev is None:
            return None
        if self._Sd is None:
            icpl, _ = local_splits(self.k)
            rows = self.cpl_of_vv[self.vv_l2g[:, icpl]]
            Sd_T = engine.unpack_sym(self.Sd_dev.cpu().numpy(), self.z["ncpl"])
            self._Sd = _assemble(len(self.vv_of_cpl), rows, self.vv_signs[:, icpl], Sd_T)
        return self._Sd

    def _ext_host(self):
        z = self.z
        E = self.ext_dev.cpu().numpy()
        ni, nc = z["n_int"], z["ncpl"]
        X = E[:, :ni * nc].reshape(-1, ni, nc)
        Sinv = engine.unpack_sym(E[:, ni * nc:], ni)
        return X, Sinv

    @property
    def ext(self):
        if self.ext_dev is None:
            return None
        return list(self._ext_host()[0])

    @property
    def soo_dense(self):
        if self.ext_dev is None:
            return None
        icpl, iint = local_splits(self.k)
        S = self.S_T_host()
        return list(S[:, iint][:, :, iint])

    @property
    def soo_chol(self):
        import scipy.linalg as sla
        if self.ext_dev is None:
            return None
        return [sla.cho_factor(s) for s in self.soo_dense]

    def _vv_codes_all(self):
        """int32 device codes over ALL (V, Vhat) dofs (2*global + (sign < 0))."""
        if getattr(self, "_codes_all", None) is None:
            m = self.maps
            self._codes_all = engine.to_dev(
                np.ascontiguousarray((2 * m.vv_l2g + (m.vv_signs < 0)).astype(np.int32)))
        return self._codes_all

    def _vector_in(self, x_full):
        torch = _torch()
        on_host = not (hasattr(x_full, "is_cuda") and x_full.is_cuda)
        x = torch.from_numpy(np.ascontiguousarray(x_full, dtype=np.float64)).cuda() \
            if on_host else x_full.contiguous()
        if x.numel() != self.fes.n_vv:
            raise ValueError(f"expected a vector over all {self.fes.n_vv} (V, Vhat) dofs")
        return x, on_host

    @_abi.nvtx("apply_S_factorized")
    def apply_S_factorized(self, x_full, stream=None):
        """S @ x over all (V, Vhat) dofs through the exact triangular
        factorisation (reference `condensation.py:104-122`), on the GPU
        (csrc/factorized.cu: per element z_o = x_o + X x_c, d_o = S_oo z_o,
        y_c = Sd_T x_c + X^T d_o, y_o = d_o).  NumPy in -> NumPy out."""
        if self.ext_dev is None:
            raise ValueError("double_schur() must be run first")
        x, on_host = self._vector_in(x_full)
        y = _torch().zeros_like(x)
        _abi.call("mcs_apply_S_factorized", self.k, self.S_dev.shape[0], _abi.ptr(self.S_dev),
                  _abi.ptr(self.ext_dev), _abi.ptr(self.Sd_dev), _abi.ptr(self._vv_codes_all()),
                  _abi.ptr(x), _abi.ptr(y), _abi.stream(stream))
        return y.cpu().numpy() if on_host else y

    @_abi.nvtx("harmonic_extend")
    def harmonic_extend(self, x_full, stream=None):
        """Energy-minimal completion of the interior bubble dofs, out_o =
        -X x_c per element (reference `condensation.py:93-102`), on the GPU."""
        if self.ext_dev is None:
            raise ValueError("double_schur() must be run first")
        x, on_host = self._vector_in(x_full)
        out = x.clone()
        _abi.call("mcs_harmonic_extend", self.k, self.S_dev.shape[0], _abi.ptr(self.ext_dev),
                  _abi.ptr(self._vv_codes_all()), _abi.ptr(x), _abi.ptr(out),
                  _abi.stream(stream))
        return out.cpu().numpy() if on_host else out

    @property
    def recovery(self):
        """Per-element R_T = M^-1 Bsig^T ((ns + nw) x nloc, reference
        `condensation.py:33,173-177`), materialised lazily on the GPU: the
        recovery kernel (csrc/recover.cu) evaluated on the nloc local unit
        vectors of every element at once (so = -R_T e_j).  The solver path
        never touches it (572 MB at cfg2)."""
        if getattr(self, "_recovery", None) is None:
            torch = _torch()
            k, nt = self.k, self.fes.mesh.num_triangles
            z = self.z
            nloc, ns, nw = z["nloc"], z["ns"], z["nw"]
            if k not in _RECOVERY:
                _RECOVERY[k] = engine.to_dev(engine.recovery_tables(self.refs))
            W = engine.to_dev(element_weights(self.fes, self.nu))
            priv = torch.arange(nt * nloc, dtype=torch.int32, device="cuda").view(nt, nloc) * 2
            R = torch.empty((nt, ns + nw, nloc), dtype=torch.float64, device="cuda")
            x = torch.zeros(nt * nloc, dtype=torch.float64, device="cuda")
            xv = x.view(nt, nloc)
            for j in range(nloc):
                xv.zero_()
                xv[:, j] = 1.0
                sig, om, info = engine.recover_stress(k, nt, W, _RECOVERY[k], priv, x)
                self.check_info(info, "singular local stress block")
                R[:, :ns, j] = -sig.view(nt, ns)
                R[:, ns:, j] = -om.view(nt, nw)
            self._recovery = list(R.cpu().numpy())
        return self._recovery

    @_abi.nvtx("recover_stress")
    def recover_stress(self, x_full, stream=None):
        """Element-wise (sigma, omega) from a velocity vector over all (V, Vhat)
        dofs (reference `condensation.py:64-74`), on the GPU
        (csrc/recover.cu).  NumPy in -> NumPy out; CUDA tensor in -> tensors."""
        torch = _torch()
        k, nt = self.k, self.fes.mesh.num_triangles
        if k not in _RECOVERY:
            _RECOVERY[k] = engine.to_dev(engine.recovery_tables(self.refs))
        if getattr(self, "_rec_inputs", None) is None:
            m = self.maps
            codes = (2 * m.vv_l2g + (m.vv_signs < 0)).astype(np.int32)
            self._rec_inputs = (engine.to_dev(element_weights(self.fes, self.nu)),
                                engine.to_dev(np.ascontiguousarray(codes)))
        W, codes = self._rec_inputs
        on_host = not (hasattr(x_full, "is_cuda") and x_full.is_cuda)
        x = torch.from_numpy(np.ascontiguousarray(x_full, dtype=np.float64)).cuda() \
            if on_host else x_full.contiguous()
        sig, om, info = engine.recover_stress(k, nt, W, _RECOVERY[k], codes, x, stream=stream)
        self.check_info(info, "singular local stress block")
        if on_host:
            return sig.cpu().numpy(), om.cpu().numpy()
        return sig, om

    def s_energy(self, x_full):
        return float(x_full @ (self.S @ x_full))

    def check_info(self, info, what, mask=None):
        v = info.cpu().numpy()
        bad = np.flatnonzero(v if mask is None else (v & mask))
        if len(bad):
            raise RuntimeError(f"{what} on element {int(bad[0])}")


_FUSED = {}
_RECOVERY = {}


def _fused_tables(k, refs):
    """Reference-cell tables of the fused kernel on the device (per k)."""
    if k not in _FUSED:
        _FUSED[k] = engine.to_dev(engine.fused_tables(refs)[0])
    return _FUSED[k]
STRUCT_TOL = 1e-10
# k = 5, 6: the double Schur as a separate warp-per-element kernel (default,
# 8.9 + 5.1 ms at cfg3) or as the last phase of the condensation kernel
# (MCS_GEN_DS=1, bitwise identical, measured 14.9 ms: its serial Cholesky
# phase idles three of the CTA's four warps next to the DMMA streams of the
# co-resident CTAs)
_GEN_DS = __import__("os").environ.get("MCS_GEN_DS", "0") == "1"


@_abi.nvtx("condense")
def condense_sigma_omega(fes, nu: float, body_force=None, blocks=None,
                         stream=None) -> CondensedSystem:
    """Eliminate (sigma, omega) element-wise on the GPU (reference
    `condensation.py:136-188`).  `blocks` (a list of ElementBlocks, as the
    reference accepts) is packed and uploaded; otherwise the blocks are
    generated on the GPU from the element geometry (refblocks.py).

    Element blocks of the MCS spaces have the block structure of DESIGN.md
    §3.2 and go through the structured kernel (S_T = adiv + Y Y^T);
    user-supplied blocks without that structure take the general dense
    signed-Cholesky kernel.  Both are GPU paths."""
    torch = _torch()
    _abi.lib()
    k = fes.k
    refs = build_refs(fes)
    nt = fes.mesh.num_triangles
    pending = None
    if blocks is not None:
        arr = lambda name: np.array([getattr(b, name) for b in blocks])
        msig, bws = arr("msig"), arr("bws")
        if engine.structure_error(msig, bws, k) <= STRUCT_TOL:
            rec_h = engine.pack_srecords(k, msig, bws, arr("bus"), arr("bhs"), arr("adiv"))
            S_dev, info = engine.condense_struct(k, engine.to_dev(rec_h), stream=stream)
        else:
            rec_h = engine.pack_records(k, msig, bws, arr("bus"), arr("bhs"), arr("adiv"))
            S_dev, info = engine.condense(k, engine.to_dev(rec_h), stream=stream)
        loads = np.array([b.load for b in blocks])
    elif k in engine.FUSED_DEGREES:
        W = engine.to_dev(element_weights(fes, nu))
        S_dev, ext, Sd, info = engine.condense_fused(k, nt, W, _fused_tables(k, refs),
                                                     stream=stream)
        pending = (ext, Sd, info)
        loads = load_vectors(fes, refs, body_force)
    elif _GEN_DS:   # k = 5, 6, MCS_GEN_DS=1: condensation + double Schur in one kernel
        W = engine.to_dev(element_weights(fes, nu))
        S_dev, ext, Sd, info = engine.condense_gen_ds(k, nt, W, _fused_tables(k, refs),
                                                      stream=stream)
        pending = (ext, Sd, info)
        loads = load_vectors(fes, refs, body_force)
    else:       # k = 5, 6: generation-fused condensation; double_schur() runs next
        W = engine.to_dev(element_weights(fes, nu))
        S_dev, info = engine.condense_gen(k, nt, W, _fused_tables(k, refs), stream=stream)
        loads = load_vectors(fes, refs, body_force)
    maps = element_maps(fes)
    load = np.zeros(fes.n_vv)
    nu_l = refs.bus_vol.shape[0]
    np.add.at(load, maps.vv_l2g[:, :nu_l].ravel(),
              (loads * maps.vv_signs[:, :nu_l]).ravel())
    sys_ = CondensedSystem(fes, nu, S_dev, load, maps, refs, None)
    sys_.check_info(info, "singular local stress block", mask=1 if pending else None)
    sys_._pending_ds = pending
    return sys_


@_abi.nvtx("double_schur")
def double_schur(sys: CondensedSystem, stream=None) -> CondensedSystem:
    """Eliminate interior bubbles per element on the GPU (reference
    `condensation.py:191-239`); mutates and returns `sys`."""
    torch = _torch()
    k = sys.k
    nt = sys.S_dev.shape[0]
    if sys._pending_ds is not None:             # computed with S_T (fused kernel)
        ext, Sd, info = sys._pending_ds
        sys._pending_ds = None
        sys.ext_dev, sys.Sd_dev = ext, Sd
        sys.vv_of_cpl, sys.cpl_of_vv = sys.maps.vv_of_cpl, sys.maps.cpl_of_vv
        sys.check_info(info, "interior velocity block not SPD", mask=2)
        return sys
    ext = torch.empty((nt, _abi.call("mcs_ext_stride", k)), dtype=torch.float64, device="cuda")
    Sd = torch.empty((nt, _abi.call("mcs_sd_stride", k)), dtype=torch.float64, device="cuda")
    info = torch.empty(nt, dtype=torch.int32, device="cuda")
    _abi.call("mcs_double_schur", k, nt, _abi.ptr(sys.S_dev), _abi.ptr(ext), _abi.ptr(Sd),
              _abi.ptr(info), _abi.stream(stream))
    sys.ext_dev, sys.Sd_dev = ext, Sd
    sys.vv_of_cpl, sys.cpl_of_vv = sys.maps.vv_of_cpl, sys.maps.cpl_of_vv
    sys.check_info(info, "interior velocity block not SPD")
    return sys
