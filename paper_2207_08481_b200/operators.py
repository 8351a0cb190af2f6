"""Device operators over free-dof vectors (C-ABI calls, stream-ordered).

`SOperator` is the matrix-free `S_free @ v` of driver.py:138-144 and
`SdOperator` the `Sd[free_cpl][:, free_cpl] @ v` of driver.py:95-96, both
evaluated element by element from the packed per-element matrices (kernel
`mcs_apply_elem`).  Callables accept torch CUDA float64
tensors (fast path) or NumPy arrays (compatibility path: H2D, apply, D2H).
"""

from __future__ import annotations

import numpy as np

from . import _abi


def torch_mod():
    import torch
    return torch


def as_device(v):
    torch = torch_mod()
    if isinstance(v, torch.Tensor):
        if not v.is_cuda or v.dtype != torch.float64:
            raise TypeError("expected a float64 CUDA tensor")
        return v.contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).cuda(), True


def empty(n):
    torch = torch_mod()
    return torch.empty(n, dtype=torch.float64, device="cuda")


class Workspace:
    """Reduction scratch + device scalar slots shared by the PCG kernels."""

    RZ0, RZ1, PAP, RR, BB, TMP = 0, 1, 2, 3, 4, 5
    PAP2, RR2, GATE, BNORM, RTOL = 6, 7, 8, 9, 10   # second step of a graphed pair
    TMP2 = 11
    GS_GATE, TMP3 = 12, 13   # GMRES: device DGKS decision, ||w||^2 after the second pass

    def __init__(self):
        torch = torch_mod()
        n = _abi.call("mcs_reduce_workspace_len")
        self.partials = torch.zeros(n, dtype=torch.float64, device="cuda")
        self.counter = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.sc = torch.zeros(16, dtype=torch.float64, device="cuda")

    def dot(self, x, y, slot, stream=None):
        _abi.call("mcs_dot", x.numel(), _abi.ptr(x), _abi.ptr(y), _abi.ptr(self.partials),
                  _abi.ptr(self.counter), self.sc.data_ptr() + 8 * slot, _abi.stream(stream))

    def dot_host(self, x, y):
        self.dot(x, y, self.TMP)
        return float(self.sc[self.TMP].item())


_WS = None


def workspace() -> Workspace:
    global _WS
    if _WS is None:
        _WS = Workspace()
    return _WS


def axpby(a, x, b, y, stream=None):
    """y = a x + b y."""
    _abi.call("mcs_axpby", y.numel(), float(a), _abi.ptr(x), float(b), _abi.ptr(y),
              _abi.stream(stream))
    return y


class _ElemOperator:
    which = 0
    graphable = True          # pure stream-ordered kernels: CUDA-graph capturable

    def __init__(self, sys_, M_dev, codes_dev, n):
        self.sys, self.k = sys_, sys_.k
        self.M, self.codes, self.n = M_dev, codes_dev, n
        self.nt = M_dev.shape[0]
        self.shape = (n, n)

    @_abi.nvtx("apply_elem")
    def apply(self, x, out=None, stream=None):
        xd, host = as_device(x)
        y = out if out is not None else empty(self.n)
        _abi.call("mcs_apply_elem", self.k, self.which, self.nt, _abi.ptr(self.M),
                  _abi.ptr(self.codes), _abi.ptr(xd), _abi.ptr(y), self.n, _abi.stream(stream))
        return y.cpu().numpy() if host else y

    __call__ = apply

    def apply_dot(self, x, out, slot, stream=None):
        """out = A x and workspace scalar `slot` = x . (A x), accumulated
        element by element inside the apply kernel (no separate dot pass)."""
        ws = workspace()
        _abi.call("mcs_apply_elem_dot", self.k, self.which, self.nt, _abi.ptr(self.M),
                  _abi.ptr(self.codes), _abi.ptr(x), _abi.ptr(out), self.n,
                  _abi.ptr(ws.partials), _abi.ptr(ws.counter), ws.sc.data_ptr() + 8 * slot,
                  _abi.stream(stream))
        return out

    def __matmul__(self, x):
        return self.apply(x)


class SOperator(_ElemOperator):
    """Condensed operator on free (V, Vhat) dofs."""
    which = 0

    def __init__(self, sys_):
        m = sys_.dev_maps()
        super().__init__(sys_, sys_.S_dev, m["vv_codes"], sys_.maps.n_vv_free)


class SdOperator(_ElemOperator):
    """Double Schur complement on free coupling dofs."""
    which = 1

    def __init__(self, sys_):
        if sys_.Sd_dev is None:
            raise ValueError("double_schur() must be run first")
        m = sys_.dev_maps()
        super().__init__(sys_, sys_.Sd_dev, m["cpl_codes"], sys_.maps.n_cpl_free)


class BOperator:
    """Divergence constraint B_free: free (V, Vhat) dofs -> pressure dofs
    (reference `sys_.B[:, vv_free]`, condensation.py:178-186; element-batched
    from the J-invariant Bpu, csrc/stokes.cu)."""

    def __init__(self, sys_):
        torch = torch_mod()
        self.sys, self.k = sys_, sys_.k
        z = sys_.z
        self.nq, self.nu, self.nloc = z["nq"], z["nu"], z["nloc"]
        self.nt = sys_.S_dev.shape[0]
        self.Bpu = torch.from_numpy(np.ascontiguousarray(sys_.refs.bpu)).cuda()
        self.codes = sys_.dev_maps()["vv_codes"]
        self.n_p = self.nt * self.nq
        self.n_v = sys_.maps.n_vv_free
        self.shape = (self.n_p, self.n_v)

    def apply(self, x, out=None, stream=None):
        xd, host = as_device(x)
        y = out if out is not None else empty(self.n_p)
        _abi.call("mcs_apply_B", self.nq, self.nu, self.nloc, self.nt, _abi.ptr(self.Bpu),
                  _abi.ptr(self.codes), _abi.ptr(xd), _abi.ptr(y), _abi.stream(stream))
        return y.cpu().numpy() if host else y

    def apply_T(self, p, out=None, stream=None):
        pd, host = as_device(p)
        y = out if out is not None else empty(self.n_v)
        _abi.call("mcs_zero", y.numel(), _abi.ptr(y), _abi.stream(stream))   # memset node
        _abi.call("mcs_apply_BT", self.nq, self.nu, self.nloc, self.nt, _abi.ptr(self.Bpu),
                  _abi.ptr(self.codes), _abi.ptr(pd), _abi.ptr(y), _abi.stream(stream))
        return y.cpu().numpy() if host else y

    __call__ = apply

    def __matmul__(self, x):
        return self.apply(x)


class SaddleOperator:
    """K = [[S_free, B_free^T], [B_free, 0]] on stacked (velocity, pressure)
    vectors (reference driver.py:150)."""

    def __init__(self, sys_):
        self.S = SOperator(sys_)
        self.B = BOperator(sys_)
        self.n_v, self.n_p = self.B.n_v, self.B.n_p
        self.n = self.n_v + self.n_p
        self.shape = (self.n, self.n)
        self._bt = empty(self.n_v)

    def apply(self, x, out=None, stream=None):
        xd, host = as_device(x)
        y = out if out is not None else empty(self.n)
        self.S.apply(xd[:self.n_v], out=y[:self.n_v], stream=stream)
        self.B.apply_T(xd[self.n_v:], out=self._bt, stream=stream)
        axpby(1.0, self._bt, 1.0, y[:self.n_v], stream)     # S x_u + (B^T x_p): fixed order
        self.B.apply(xd[:self.n_v], out=y[self.n_v:], stream=stream)
        return y.cpu().numpy() if host else y

    __call__ = apply

    def __matmul__(self, x):
        return self.apply(x)
