"""Element -> free-dof index maps for the GPU operators (host setup).

All GPU vectors of the PCG live in the reference's free-dof numbering
(`fes.vv_free`, `CondensedSystem.free_mask_cpl()`), so results are directly
comparable with `S_free @ v` (driver.py:138) and the reference
preconditioner.  Per element the kernels read int32 *codes*:
`code = 2*free_index + (sign < 0)`, or -1 for a constrained dof.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .refblocks import local_sizes


def local_splits(k: int):
    """(icpl, iint): local coupling / bubble positions (condensation.py:124-133)."""
    z = local_sizes(k)
    icpl = np.concatenate([np.arange(z["n_em"]), np.arange(z["nu"], z["nloc"])])
    return icpl, np.arange(z["n_em"], z["nu"])


def free_index(mask: np.ndarray) -> np.ndarray:
    idx = -np.ones(len(mask), dtype=np.int64)
    idx[mask] = np.arange(int(mask.sum()))
    return idx


def codes(idx: np.ndarray, signs: np.ndarray) -> np.ndarray:
    return np.where(idx >= 0, 2 * idx + (signs < 0), -1).astype(np.int32)


@dataclass
class ElementMaps:
    vv_l2g: np.ndarray          # (nt, nloc) combined local -> global vv
    vv_signs: np.ndarray        # (nt, nloc)
    vv_codes: np.ndarray        # (nt, nloc) int32 over vv-free
    bubble_idx: np.ndarray      # (nt, n_int) int32 vv-free index of bubbles
    cpl_codes: np.ndarray       # (nt, ncpl) int32 over cpl-free
    vv_of_cpl: np.ndarray       # cpl -> vv
    cpl_of_vv: np.ndarray       # vv -> cpl or -1
    free_cpl: np.ndarray        # bool over cpl
    cplfree_to_vvfree: np.ndarray  # int32 (n_cpl_free,)
    n_vv_free: int
    n_cpl_free: int


def element_maps(fes) -> ElementMaps:
    k = fes.k
    l2g = np.concatenate([fes.dof_v.loc2glob, fes.n_v + fes.dof_vhat.loc2glob], 1)
    sg = np.concatenate([fes.dof_v.signs, fes.dof_vhat.signs], 1)
    fvv = free_index(fes.vv_free)
    icpl, iint = local_splits(k)
    mask_cpl = ~fes.vv_interior
    vv_of_cpl = np.flatnonzero(mask_cpl)
    cpl_of_vv = -np.ones(fes.n_vv, dtype=np.int64)
    cpl_of_vv[mask_cpl] = np.arange(mask_cpl.sum())
    free_cpl = fes.vv_free[vv_of_cpl]
    fcp = free_index(free_cpl)
    cp_idx = fcp[cpl_of_vv[l2g[:, icpl]]]
    bub = fvv[l2g[:, iint]]
    if np.any(bub < 0):
        raise ValueError("interior bubble dofs must be free")
    return ElementMaps(
        vv_l2g=l2g, vv_signs=sg, vv_codes=codes(fvv[l2g], sg),
        bubble_idx=bub.astype(np.int32), cpl_codes=codes(cp_idx, sg[:, icpl]),
        vv_of_cpl=vv_of_cpl, cpl_of_vv=cpl_of_vv, free_cpl=free_cpl,
        cplfree_to_vvfree=fvv[vv_of_cpl[free_cpl]].astype(np.int32),
        n_vv_free=int(fes.vv_free.sum()), n_cpl_free=int(free_cpl.sum()))


def facet_slots(fes, maps: ElementMaps):
    """Facet blocks of S_d (preconditioners.py:266-280): one per facet with at
    least one free coupling dof, in facet order.  Returns (slots (nb, 4) int32
    = (t0, le0, t1, le1), facet ids)."""
    m, k = fes.mesh, fes.k
    nt = m.num_triangles
    tf = m.tri_facets
    t_idx = np.repeat(np.arange(nt), 3)
    le_idx = np.tile(np.arange(3), nt)
    f_idx = tf.ravel()
    order = np.lexsort((t_idx, f_idx))
    f_s, t_s, le_s = f_idx[order], t_idx[order], le_idx[order]
    first = np.r_[True, f_s[1:] != f_s[:-1]]
    nf = m.num_facets
    slots = -np.ones((nf, 4), dtype=np.int64)
    slots[f_s[first], 0] = t_s[first]
    slots[f_s[first], 1] = le_s[first]
    slots[f_s[~first], 2] = t_s[~first]
    slots[f_s[~first], 3] = le_s[~first]
    # a facet block exists iff one of its (k+1) normal or k tangential dofs is free
    fdofs_n = np.arange(nf)[:, None] * (k + 1) + np.arange(k + 1)
    fdofs_t = fes.n_v + np.arange(nf)[:, None] * k + np.arange(k)
    has = fes.vv_free[fdofs_n].any(1) | fes.vv_free[fdofs_t].any(1)
    fid = np.flatnonzero(has)
    return slots[fid].astype(np.int32), fid
