"""CPU: the C-ABI library loads and exports every symbol include/stam_cuda.h
declares (no compute calls without a GPU)."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1802_10574_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "stam_cuda.h").read_text()
    return sorted(set(re.findall(r"STAM_CUDA_API\s+[\w\s\*]+?\b(stam_cuda_\w+)\s*\(", text)))


def test_header_declares_the_kernel_calls():
    syms = declared_symbols()
    for name in ("stam_cuda_spgemm", "stam_cuda_spadd", "stam_cuda_mttkrp_dense",
                 "stam_cuda_mttkrp_sparse", "stam_cuda_ctx_create", "stam_cuda_release"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(N.library_path()))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(N.SIGNATURES) == set(declared_symbols())


def test_abi_version_and_defaults():
    lib = N.load()
    assert lib.stam_cuda_abi_version() == 1
    o = N.Options()
    lib.stam_cuda_default_options(C.byref(o))
    assert (o.sort, o.mode, o.result_mem, o.timing) == (1, 0, N.STAM_MEM_DEVICE, 0)


def test_struct_layouts_match_header_sizes():
    # 64-bit fields first, 8-byte aligned; views/results as declared
    assert C.sizeof(N.CsrView) == 56
    assert C.sizeof(N.Csf3View) == 88
    assert C.sizeof(N.DenseView) == 32
    assert C.sizeof(N.CsrResult) == 64
    assert C.sizeof(N.Options) == 16


def test_no_device_is_an_error_not_a_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    status = N.load().stam_cuda_ctx_create(0, C.byref(h))
    assert status == 66  # STAM_ERR_NO_DEVICE
    assert b"device" in N.load().stam_cuda_last_error().lower()


def test_error_codes_mirror_reference_enum():
    # 1 + (int)stam::ErrorCode, include/stam/error.h
    assert N.ERROR_CODES[2] == "DimensionMismatch" and N.ERROR_CODES[14] == "UnsupportedMerge"
    e = N.StamError(3, "x")
    assert e.code == "DimensionMismatch"
