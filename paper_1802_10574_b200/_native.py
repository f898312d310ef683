"""ctypes binding of the C ABI in ``include/stam_cuda.h``.

The structures below mirror the header field for field.  Loading fails loudly
when ``_lib/libstam_cuda.so`` is missing: there is no CPU fallback anywhere on
the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

_LIB_DIR = Path(__file__).resolve().parent / "_lib"

STAM_OK = 0
STAM_MEM_HOST = 0
STAM_MEM_DEVICE = 1
STAM_MODE_FUSED, STAM_MODE_ASSEMBLE, STAM_MODE_COMPUTE = 0, 1, 2

# reference ErrorCode names (include/stam/error.h:9-31), index = status - 1
ERROR_CODES = [
    "Parse", "ArityMismatch", "DimensionMismatch", "OrderMismatch", "OutOfRange",
    "AppendOutOfOrder", "IllFormed", "PreconditionViolated", "SequencePresent",
    "DistributivityViolated", "VariableNotInScope", "ReusePrecondition1",
    "ReusePrecondition2", "NeedsReorder", "UnsupportedMerge", "UnplannableResult",
    "MissingBinding", "MissingSlot", "CheckFailed", "Io", "Internal",
]
DEVICE_CODES = {64: "Cuda", 65: "OutOfMemory", 66: "NoDevice"}

P64 = C.POINTER(C.c_int64)
PD = C.POINTER(C.c_double)


class CsrView(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("pos", C.c_void_p), ("idx", C.c_void_p), ("vals", C.c_void_p),
                ("mem", C.c_int32), ("_pad", C.c_int32)]


class Csf3View(C.Structure):
    _fields_ = [("dims", C.c_int64 * 3), ("nfibers", C.c_int64), ("nnz", C.c_int64),
                ("pos1", C.c_void_p), ("idx1", C.c_void_p), ("pos2", C.c_void_p),
                ("idx2", C.c_void_p), ("vals", C.c_void_p),
                ("mem", C.c_int32), ("_pad", C.c_int32)]


class DenseView(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("vals", C.c_void_p),
                ("mem", C.c_int32), ("_pad", C.c_int32)]


class CsrResult(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("pos", C.c_void_p), ("idx", C.c_void_p), ("vals", C.c_void_p),
                ("mem", C.c_int32), ("_pad", C.c_int32), ("handle", C.c_void_p)]


class DenseResult(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("vals", C.c_void_p),
                ("mem", C.c_int32), ("_pad", C.c_int32), ("handle", C.c_void_p)]


class Options(C.Structure):
    _fields_ = [("sort", C.c_int32), ("mode", C.c_int32), ("result_mem", C.c_int32),
                ("timing", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("mults", C.c_int64), ("adds", C.c_int64), ("merge_compares", C.c_int64),
                ("sparse_inserts", C.c_int64), ("appends", C.c_int64),
                ("ws_inserts", C.c_int64), ("ws_resets", C.c_int64),
                ("bytes_allocated", C.c_int64), ("kernel_launches", C.c_int64),
                ("main_kernel_ms", C.c_float), ("total_kernel_ms", C.c_float),
                ("h2d_ms", C.c_float), ("d2h_ms", C.c_float),
                ("main_kernel", C.c_char * 48)]

    def as_dict(self) -> dict:
        d = {name: getattr(self, name) for name, _ in self._fields_}
        d["main_kernel"] = self.main_kernel.decode()
        return d


# Every symbol include/stam_cuda.h declares, with its signature.
SIGNATURES = {
    "stam_cuda_abi_version": (C.c_int, []),
    "stam_cuda_last_error": (C.c_char_p, []),
    "stam_cuda_default_options": (None, [C.POINTER(Options)]),
    "stam_cuda_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "stam_cuda_ctx_destroy": (C.c_int, [C.c_void_p]),
    "stam_cuda_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "stam_cuda_ctx_device": (C.c_int, [C.c_void_p]),
    "stam_cuda_synchronize": (C.c_int, [C.c_void_p]),
    "stam_cuda_release": (C.c_int, [C.c_void_p, C.c_void_p]),
    "stam_cuda_spgemm": (C.c_int, [C.c_void_p, C.POINTER(CsrView), C.POINTER(CsrView),
                                   C.POINTER(Options), C.POINTER(CsrResult), C.POINTER(Stats)]),
    "stam_cuda_spgemm_compute": (C.c_int, [C.c_void_p, C.POINTER(CsrView), C.POINTER(CsrView),
                                           C.POINTER(CsrView), C.POINTER(Options),
                                           C.POINTER(CsrResult), C.POINTER(Stats)]),
    "stam_cuda_spadd": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(CsrView),
                                  C.POINTER(Options), C.POINTER(CsrResult), C.POINTER(Stats)]),
    "stam_cuda_spadd_compute": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(CsrView),
                                          C.POINTER(CsrView), C.POINTER(Options),
                                          C.POINTER(CsrResult), C.POINTER(Stats)]),
    "stam_cuda_mttkrp_dense": (C.c_int, [C.c_void_p, C.POINTER(Csf3View), C.POINTER(DenseView),
                                         C.POINTER(DenseView), C.POINTER(Options),
                                         C.POINTER(DenseResult), C.POINTER(Stats)]),
    "stam_cuda_mttkrp_sparse": (C.c_int, [C.c_void_p, C.POINTER(Csf3View), C.POINTER(CsrView),
                                          C.POINTER(CsrView), C.POINTER(Options),
                                          C.POINTER(CsrResult), C.POINTER(Stats)]),
    "stam_cuda_ttv": (C.c_int, [C.c_void_p, C.POINTER(Csf3View), C.POINTER(DenseView),
                                C.POINTER(Options), C.POINTER(CsrResult), C.POINTER(Stats)]),
    "stam_cuda_rowdot": (C.c_int, [C.c_void_p, C.POINTER(CsrView), C.POINTER(CsrView),
                                   C.POINTER(Options), C.POINTER(DenseResult), C.POINTER(Stats)]),
    "stam_cuda_spadd_merge": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(CsrView),
                                        C.POINTER(Options), C.POINTER(CsrResult),
                                        C.POINTER(Stats)]),
}

_lock = threading.Lock()
_lib = None


class StamError(RuntimeError):
    """Mirror of ``stam::Error``: carries the reference ``ErrorCode`` name."""

    def __init__(self, status: int, message: str):
        self.status = status
        if 1 <= status <= len(ERROR_CODES):
            self.code = ERROR_CODES[status - 1]
        else:
            self.code = DEVICE_CODES.get(status, f"Status{status}")
        super().__init__(f"{self.code}: {message}")


def library_path() -> Path:
    # STAM_CUDA_LIB: an alternative build of the same library (tuning variants)
    alt = os.environ.get("STAM_CUDA_LIB")
    return Path(alt) if alt else _LIB_DIR / "libstam_cuda.so"


def load() -> C.CDLL:
    """Loads libstam_cuda.so; raises if it was not built (no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if not path.exists():
            raise ImportError(
                f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the sm_100a kernels have no CPU fallback)")
        lib = C.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.stam_cuda_abi_version() != 1:
            raise ImportError("libstam_cuda.so ABI version mismatch")
        _lib = lib
        return lib


def check(status: int) -> None:
    if status != STAM_OK:
        msg = load().stam_cuda_last_error()
        raise StamError(status, msg.decode() if msg else "")
