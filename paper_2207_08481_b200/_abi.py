"""ctypes binding of the C ABI in `include/mcs_abi.h` (libmcsgpu.so).

Every entry point takes device pointers owned by the caller (torch tensors)
and a `cudaStream_t`; calls are asynchronous on that stream.  Return codes:
0 ok, <0 CUDA / argument error, >0 first failing element (1-based).  There is
deliberately NO fallback: if the library is missing or a call fails, the
product path raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmcsgpu.so")

_p, _i, _l, _d = C.c_void_p, C.c_int, C.c_int64, C.c_double

# name -> argtypes (restype int).  Mirrors include/mcs_abi.h one to one.
SIGNATURES = {
    # condense.cu
    "mcs_spd_schur_batched": [_i, _i, _l, _p, _p, _p, _p, _p],
    "mcs_record_len": [_i],
    "mcs_st_stride": [_i],
    "mcs_condense": [_i, _l, _p, _p, _p, _p],
    "mcs_element_blocks": [_l, _i, _p, _i, _p, _p, _p, _p, _p],
    # condense_struct.cu
    "mcs_srec_len": [_i],
    "mcs_condense_struct": [_i, _l, _p, _p, _p, _p],
    "mcs_condense_gen": [_i, _l, _p, _i, _p, _p, _p, _p],
    "mcs_condense_gen_ds": [_i, _l, _p, _i, _p, _p, _p, _p, _p, _p],
    # stokes.cu
    "mcs_apply_B": [_i, _i, _i, _l, _p, _p, _p, _p, _p],
    "mcs_apply_BT": [_i, _i, _i, _l, _p, _p, _p, _p, _p],
    "mcs_mdot_len": [],
    "mcs_mdot": [_i, _l, _l, _p, _p, _p, _p, _p],
    "mcs_gemv_acc": [_i, _l, _l, _p, _p, _d, _d, _p, _p],
    "mcs_mdot_gated": [_i, _l, _l, _p, _p, _p, _p, _p, _p],
    "mcs_gemv_acc_gated": [_i, _l, _l, _p, _p, _d, _d, _p, _p, _p],
    "mcs_gs_gate": [_p, _i, _i, _i, _p],
    "mcs_gs_fused_blocks": [],
    "mcs_gs_fused": [_i, _l, _l, _p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _p],
    # postcheck.cu
    "mcs_post_checks": [_l, _i, _i, _p, _p, _p, _p, _p, _p, _i, _i, _i, _p, _p, _p, _p, _p, _p,
                        _p, _i, _p],
    # recover.cu
    "mcs_recover_table_len": [_i],
    "mcs_recover_stress": [_i, _l, _p, _i, _p, _p, _p, _p, _p, _p, _p],
    # condense_fused.cu
    "mcs_fused_table_len": [_i],
    "mcs_condense_fused": [_i, _l, _p, _i, _p, _p, _p, _p, _p, _p],
    # double_schur.cu
    "mcs_ext_stride": [_i],
    "mcs_sd_stride": [_i],
    "mcs_double_schur": [_i, _l, _p, _p, _p, _p, _p],
    # apply.cu
    "mcs_apply_elem": [_i, _i, _l, _p, _p, _p, _p, _l, _p],
    "mcs_apply_elem_dot": [_i, _i, _l, _p, _p, _p, _p, _l, _p, _p, _p, _p],
    "mcs_ext_restrict": [_i, _l, _p, _p, _p, _p, _p, _p, _l, _p],
    "mcs_ext_prolong": [_i, _l, _p, _p, _p, _p, _p, _p, _p, _p],
    "mcs_gather_sub": [_i, _p, _p, _p, _p, _p],
    "mcs_scatter": [_i, _p, _p, _p, _p],
    # precond.cu
    "mcs_jacobi_setup": [_i, _i, _p, _i, _p, _p, _p, _p, _p, _p, _p],
    "mcs_jacobi_apply": [_i, _i, _p, _p, _p, _p, _d, _p],
    "mcs_csr_spmv": [_i, _p, _p, _p, _p, _p, _d, _d, _i, _p],
    "mcs_dense_gemv": [_i, _p, _p, _p, _p],
    # coarse.cu
    "mcs_mf_forward": [_i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i, _i, _p],
    "mcs_mf_backward": [_i, _p, _p, _p, _p, _p, _p, _p, _p, _i, _i, _p],
    "mcs_mf_top_ld": [_i],
    "mcs_mf_top": [_i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p],
    # blas1.cu
    "mcs_reduce_workspace_len": [],
    "mcs_dot": [_l, _p, _p, _p, _p, _p, _p],
    "mcs_cg_update": [_l, _p, _p, _p, _p, _p, _i, _i, _i, _p, _p, _p],
    "mcs_cg_update_gated": [_l, _p, _p, _p, _p, _p, _i, _i, _i, _i, _i, _i, _i, _p, _p, _p],
    "mcs_xpby": [_l, _p, _p, _p, _i, _i, _p],
    "mcs_axpby": [_l, _d, _p, _d, _p, _p],
    "mcs_vdiv": [_l, _p, _p, _p, _p],
    "mcs_zero": [_l, _p, _p],
    # pcg_loop.cu
    "mcs_pcg_loop_build": [_p, _p, _p, _i, _i, _i, _i, _i, _i, _i, _p],
    "mcs_pcg_loop_launch": [_p, _p, _i, _p],
    "mcs_pcg_loop_destroy": [_p],
    # factorized.cu
    "mcs_apply_S_factorized": [_i, _l, _p, _p, _p, _p, _p, _p, _p],
    "mcs_harmonic_extend": [_i, _l, _p, _p, _p, _p, _p],
    "mcs_block_inverse": [_i, _i, _p, _p, _p, _p, _p, _p, _p],
}

_lib = None


class McsError(RuntimeError):
    pass


def lib():
    """Load libmcsgpu.so (raises if it is missing: no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise McsError(f"{LIB_PATH} missing: run `python -m "
                           "paper_2207_08481_b200.build` (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        _lib = L
    return _lib


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise McsError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise McsError("expected a contiguous tensor")
    return t.data_ptr()


def stream(s=None) -> int:
    import torch
    s = s if s is not None else torch.cuda.current_stream()
    return s.cuda_stream


def call(name, *args):
    rc = getattr(lib(), name)(*args)
    if rc < 0:
        raise McsError(f"{name} failed with CUDA error {-rc}"
                       if rc > -1000 else f"{name}: unsupported arguments ({rc})")
    return rc


# ---- NVTX ranges per kernel group: one range per public call
# (condensation, operator applies, preconditioner stages, Krylov solves) so
# Nsight timelines / `ncu --nvtx --nvtx-include` can select a group.
# MCS_NVTX=0 turns them off.  Inside a CUDA-graph replay no Python runs, so
# the ranges cost nothing on the captured PCG loop.
_NVTX = os.environ.get("MCS_NVTX", "1") != "0"


class nvtx:
    """Context manager / decorator: an NVTX range named `mcs:<name>`."""

    def __init__(self, name):
        self.name = "mcs:" + name

    def __enter__(self):
        if _NVTX:
            import torch
            torch.cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *exc):
        if _NVTX:
            import torch
            torch.cuda.nvtx.range_pop()
        return False

    def __call__(self, fn):
        import functools

        @functools.wraps(fn)
        def wrapped(*a, **kw):
            with self:
                return fn(*a, **kw)
        return wrapped
