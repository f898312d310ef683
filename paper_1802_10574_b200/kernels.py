"""Python entry points of the hot path, mirroring the C++ ``stam::spgemm`` /
``stam::spadd`` / ``stam::mttkrp`` declared in ``include/stam/kernels.h`` (the
engine slot the reference leaves empty: ``src/engine.cpp:1``; SPEC
``execute`` ``SPEC.md:377-385``).

Every call goes through the C ABI (``include/stam_cuda.h``) into the sm_100a
kernels of ``_lib/libstam_cuda.so``.  Inputs may be host arrays (numpy / CPU
torch; staged to the device inside the call) or CUDA torch tensors.  Results
are returned on the device (zero-copy torch tensors over library-owned memory)
or on the host (``result="host"``: numpy copies).  Errors raise
``StamError`` carrying the reference ``ErrorCode`` name.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .storage import CSF3, CSR, Dense


class _Owner:
    """Releases one library-owned result when the last view of it dies."""

    def __init__(self, ctx: "Context", handle: int):
        self.ctx = ctx
        self.handle = handle

    def __del__(self):
        try:
            if self.handle and self.ctx._ctx:
                # free in order after torch work already queued on the stream
                # the caller is using (results are read through torch tensors)
                self.ctx._follow_torch()
                N.load().stam_cuda_release(self.ctx._ctx, C.c_void_p(self.handle))
        except Exception:
            pass
        self.handle = 0


class _DevArray:
    """__cuda_array_interface__ over library memory (keeps its owner alive)."""

    def __init__(self, ptr: int, n: int, typestr: str, owner: _Owner):
        self._owner = owner
        self.__cuda_array_interface__ = {
            "shape": (n,), "typestr": typestr, "data": (ptr if n else 0, False),
            "version": 3, "strides": None,
        }


def _dev_tensor(ptr: int, n: int, dtype: str, owner: _Owner):
    import torch

    if n == 0:
        return torch.empty(0, dtype=getattr(torch, dtype), device="cuda")
    typestr = {"int64": "<i8", "float64": "<f8"}[dtype]
    t = torch.as_tensor(_DevArray(ptr, n, typestr, owner), device="cuda")
    t._stam_owner = owner  # noqa: SLF001 — keep the allocation alive with the tensor
    return t


def _host_copy(ptr: int, n: int, dtype) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=dtype)
    ctype = C.c_int64 if dtype == np.int64 else C.c_double
    buf = (ctype * n).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype).copy()


class Context:
    """One device + stream + memory pool (``stam_cuda_ctx``).

    Stream ordering: unless ``set_stream`` pins a stream, every call (and every
    release of a device result) runs on torch's *current* stream of the
    context's device, so CUDA-tensor inputs produced by queued torch kernels
    are complete before the library reads them, and a result's memory goes
    back to the pool only after torch work queued on that stream."""

    def __init__(self, device: int = 0):
        self._lib = N.load()
        h = C.c_void_p()
        N.check(self._lib.stam_cuda_ctx_create(int(device), C.byref(h)))
        self._ctx = h
        self.device = device
        self._pinned_stream = False
        self._cur_stream = None

    def _follow_torch(self) -> None:
        if self._pinned_stream or not self._ctx:
            return
        import sys

        torch = sys.modules.get("torch")
        if torch is None or not torch.cuda.is_initialized():
            return
        raw = int(torch.cuda.current_stream(self.device).cuda_stream)
        if raw == 0:
            raw = 1  # torch's default stream is the legacy stream (cudaStreamLegacy)
        if raw != self._cur_stream:
            N.check(self._lib.stam_cuda_ctx_set_stream(self._ctx, C.c_void_p(raw)))
            self._cur_stream = raw

    def close(self) -> None:
        if self._ctx:
            N.check(self._lib.stam_cuda_ctx_destroy(self._ctx))
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream) -> None:
        """Run on a torch.cuda.Stream (or a raw cudaStream_t int); None resets."""
        raw = 0 if stream is None else int(getattr(stream, "cuda_stream", stream))
        N.check(self._lib.stam_cuda_ctx_set_stream(self._ctx, C.c_void_p(raw)))
        self._pinned_stream = stream is not None
        self._cur_stream = raw if stream is not None else None

    def synchronize(self) -> None:
        N.check(self._lib.stam_cuda_synchronize(self._ctx))

    # -- helpers -------------------------------------------------------------
    @staticmethod
    def options(sort: bool = True, result: str = "device", timing: bool = False,
                mode: int = N.STAM_MODE_FUSED) -> N.Options:
        if result not in ("device", "host"):
            raise ValueError("result must be 'device' or 'host'")
        return N.Options(1 if sort else 0, mode,
                         N.STAM_MEM_HOST if result == "host" else N.STAM_MEM_DEVICE,
                         1 if timing else 0)

    def _csr_out(self, r: N.CsrResult) -> CSR:
        owner = _Owner(self, r.handle)
        if r.mem == N.STAM_MEM_DEVICE:
            return CSR(r.nrows, r.ncols, _dev_tensor(r.pos, r.nrows + 1, "int64", owner),
                       _dev_tensor(r.idx, r.nnz, "int64", owner),
                       _dev_tensor(r.vals, r.nnz, "float64", owner))
        out = CSR(r.nrows, r.ncols, _host_copy(r.pos, r.nrows + 1, np.int64),
                  _host_copy(r.idx, r.nnz, np.int64), _host_copy(r.vals, r.nnz, np.float64))
        del owner  # host copies made; release the pinned buffer now
        return out

    def _dense_out(self, r: N.DenseResult) -> Dense:
        owner = _Owner(self, r.handle)
        n = r.nrows * r.ncols
        if r.mem == N.STAM_MEM_DEVICE:
            return Dense(_dev_tensor(r.vals, n, "float64", owner).view(r.nrows, r.ncols))
        out = Dense(_host_copy(r.vals, n, np.float64).reshape(r.nrows, r.ncols))
        del owner
        return out

    # -- kernels -------------------------------------------------------------
    def spgemm(self, A: CSR, B: CSR, *, sort: bool = True, result: str = "device",
               timing: bool = False, stats: Optional[N.Stats] = None,
               mode: str = "fused") -> CSR:
        """mode "fused" (index + values) or "assemble" (exact index, zero
        values: the symbolic phase); see spgemm_compute for "compute"."""
        r = N.CsrResult()
        st = stats if stats is not None else N.Stats()
        opts = self.options(sort, result, timing, self._MODES[mode])
        self._follow_torch()
        N.check(self._lib.stam_cuda_spgemm(self._ctx, C.byref(A.view()), C.byref(B.view()),
                                           C.byref(opts), C.byref(r), C.byref(st)))
        return self._csr_out(r)

    def spgemm_compute(self, A: CSR, B: CSR, index: CSR, *, sort: bool = True,
                       result: str = "device", timing: bool = False,
                       stats: Optional[N.Stats] = None) -> CSR:
        """Values of A·B written into a pre-assembled index (e.g. an
        ``spgemm(..., mode="assemble")`` result): SPEC's compute-after-assemble.
        ``sort=False`` when the index rows are not sorted."""
        r = N.CsrResult()
        st = stats if stats is not None else N.Stats()
        opts = self.options(sort, result, timing, N.STAM_MODE_COMPUTE)
        self._follow_torch()
        N.check(self._lib.stam_cuda_spgemm_compute(
            self._ctx, C.byref(A.view()), C.byref(B.view()), C.byref(index.view()),
            C.byref(opts), C.byref(r), C.byref(st)))
        return self._csr_out(r)

    _MODES = {"fused": N.STAM_MODE_FUSED, "assemble": N.STAM_MODE_ASSEMBLE,
              "compute": N.STAM_MODE_COMPUTE}

    def spadd(self, ops: Sequence[CSR], *, sort: bool = True, result: str = "device",
              timing: bool = False, stats: Optional[N.Stats] = None,
              mode: str = "fused") -> CSR:
        """mode "fused" or "assemble" (exact union index, zero values)."""
        views = (N.CsrView * len(ops))(*[o.view() for o in ops])
        r = N.CsrResult()
        st = stats if stats is not None else N.Stats()
        opts = self.options(sort, result, timing, self._MODES[mode])
        self._follow_torch()
        N.check(self._lib.stam_cuda_spadd(self._ctx, len(ops), views, C.byref(opts), C.byref(r),
                                          C.byref(st)))
        return self._csr_out(r)

    def spadd_compute(self, ops: Sequence[CSR], index: CSR, *, sort: bool = True,
                      result: str = "device", timing: bool = False,
                      stats: Optional[N.Stats] = None) -> CSR:
        """Operand values written into a pre-assembled index (compute mode)."""
        views = (N.CsrView * len(ops))(*[o.view() for o in ops])
        r = N.CsrResult()
        st = stats if stats is not None else N.Stats()
        opts = self.options(sort, result, timing, N.STAM_MODE_COMPUTE)
        self._follow_torch()
        N.check(self._lib.stam_cuda_spadd_compute(self._ctx, len(ops), views,
                                                  C.byref(index.view()), C.byref(opts),
                                                  C.byref(r), C.byref(st)))
        return self._csr_out(r)

    # -- SPEC kernels outside the workspace plans ------------------------------
    def ttv(self, B: CSF3, c, *, result: str = "device", timing: bool = False,
            stats: Optional[N.Stats] = None) -> CSR:
        """A(i,j) = sum_k B(i,j,k) c(k): CSR over B's (i,j) fibers."""
        cv = c if isinstance(c, Dense) else Dense(c.reshape(-1, 1) if hasattr(c, "reshape") else c)
        r = N.CsrResult()
        st = stats if stats is not None else N.Stats()
        opts = self.options(True, result, timing)
        self._follow_torch()
        N.check(self._lib.stam_cuda_ttv(self._ctx, C.byref(B.view()), C.byref(cv.view()),
                                        C.byref(opts), C.byref(r), C.byref(st)))
        return self._csr_out(r)

    def rowdot(self, B: CSR, Cm: CSR, *, result: str = "device", timing: bool = False,
               stats: Optional[N.Stats] = None) -> Dense:
        """a(i) = sum_j B(i,j) C(i,j) (two-way intersection, no workspace)."""
        r = N.DenseResult()
        st = stats if stats is not None else N.Stats()
        opts = self.options(True, result, timing)
        self._follow_torch()
        N.check(self._lib.stam_cuda_rowdot(self._ctx, C.byref(B.view()), C.byref(Cm.view()),
                                           C.byref(opts), C.byref(r), C.byref(st)))
        return self._dense_out(r)

    def spadd_merge(self, ops: Sequence[CSR], *, result: str = "device", timing: bool = False,
                    stats: Optional[N.Stats] = None) -> CSR:
        """Merge-based SpAdd baseline: pairwise two-way unions."""
        views = (N.CsrView * len(ops))(*[o.view() for o in ops])
        r = N.CsrResult()
        st = stats if stats is not None else N.Stats()
        opts = self.options(True, result, timing)
        self._follow_torch()
        N.check(self._lib.stam_cuda_spadd_merge(self._ctx, len(ops), views, C.byref(opts),
                                                C.byref(r), C.byref(st)))
        return self._csr_out(r)

    def mttkrp(self, B: CSF3, Cf, Df, *, result: str = "device", timing: bool = False,
               stats: Optional[N.Stats] = None):
        """Dense factors (``Dense``) give a dense A; CSR factors give a CSR A."""
        st = stats if stats is not None else N.Stats()
        opts = self.options(True, result, timing)
        if isinstance(Cf, Dense) and isinstance(Df, Dense):
            r = N.DenseResult()
            self._follow_torch()
            N.check(self._lib.stam_cuda_mttkrp_dense(
                self._ctx, C.byref(B.view()), C.byref(Cf.view()), C.byref(Df.view()),
                C.byref(opts), C.byref(r), C.byref(st)))
            return self._dense_out(r)
        if isinstance(Cf, CSR) and isinstance(Df, CSR):
            r = N.CsrResult()
            self._follow_torch()
            N.check(self._lib.stam_cuda_mttkrp_sparse(
                self._ctx, C.byref(B.view()), C.byref(Cf.view()), C.byref(Df.view()),
                C.byref(opts), C.byref(r), C.byref(st)))
            return self._csr_out(r)
        raise N.StamError(8, "mttkrp factors must both be Dense or both be CSR")


_default: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def spgemm(A: CSR, B: CSR, **kw) -> CSR:
    return default_context().spgemm(A, B, **kw)


def spadd(ops: Sequence[CSR], **kw) -> CSR:
    return default_context().spadd(ops, **kw)


def mttkrp(B: CSF3, Cf, Df, **kw):
    return default_context().mttkrp(B, Cf, Df, **kw)
