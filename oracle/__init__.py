"""ctypes wrappers of the parity checkers — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py (cpu_baseline and
``--impl reference``) import this module.  It is never used by the product
path, which has no CPU fallback.

* ``port``      — ``oracle/liboracle.so``: the C restatement (stam_oracle.c),
                  with the absolute-value twin for the scaled tolerance.
* ``reference`` — ``oracle/_ref/libstamref.so``: the same loop nests run through
                  the reference's own ``stam::Workspace`` / ``TensorBuilder``
                  (compiled from /root/reference sources by oracle/Makefile).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
P64 = C.POINTER(C.c_int64)
PD = C.POINTER(C.c_double)


class OCsr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("pos", P64), ("idx", P64), ("vals", PD), ("absv", PD)]


class OCsrIn(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("pos", P64), ("idx", P64), ("vals", PD)]


class OCsf3(C.Structure):
    _fields_ = [("dims", C.c_int64 * 3), ("nfibers", C.c_int64), ("nnz", C.c_int64),
                ("pos1", P64), ("idx1", P64), ("pos2", P64), ("idx2", P64), ("vals", PD)]


class RCsrOut(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("pos", P64), ("idx", P64), ("vals", PD)]


class Counters(C.Structure):
    _fields_ = [("mults", C.c_int64), ("adds", C.c_int64), ("ws_inserts", C.c_int64),
                ("ws_resets", C.c_int64), ("appends", C.c_int64), ("merge_compares", C.c_int64)]


_port = None
_ref = None


def port_lib():
    global _port
    if _port is None:
        path = HERE / "liboracle.so"
        if not path.exists():
            raise ImportError(f"{path} missing; run `make -C oracle`")
        lib = C.CDLL(str(path))
        lib.oracle_spgemm.argtypes = [C.POINTER(OCsrIn), C.POINTER(OCsrIn), C.c_int,
                                      C.POINTER(OCsr)]
        lib.oracle_spadd.argtypes = [C.c_int, C.POINTER(OCsrIn), C.c_int, C.POINTER(OCsr)]
        lib.oracle_mttkrp_dense.argtypes = [C.POINTER(OCsf3), PD, PD, C.c_int64, C.c_int, PD, PD]
        lib.oracle_mttkrp_sparse.argtypes = [C.POINTER(OCsf3), C.POINTER(OCsrIn),
                                             C.POINTER(OCsrIn), C.c_int, C.POINTER(OCsr)]
        lib.oracle_ttv.argtypes = [C.POINTER(OCsf3), PD, C.POINTER(OCsr)]
        lib.oracle_rowdot.argtypes = [C.POINTER(OCsrIn), C.POINTER(OCsrIn), PD, PD]
        lib.oracle_spadd_merge.argtypes = [C.c_int, C.POINTER(OCsrIn), C.POINTER(OCsr)]
        lib.oracle_free.argtypes = [C.POINTER(OCsr)]
        lib.oracle_last_counters.argtypes = [C.POINTER(Counters)]
        _port = lib
    return _port


def ref_available() -> bool:
    return (HERE / "_ref" / "libstamref.so").exists()


def ref_lib():
    global _ref
    if _ref is None:
        path = HERE / "_ref" / "libstamref.so"
        if not path.exists():
            raise ImportError(f"{path} missing (built from /root/reference by oracle/Makefile)")
        lib = C.CDLL(str(path))
        lib.ref_spgemm.argtypes = [C.POINTER(OCsrIn), C.POINTER(OCsrIn), C.c_int,
                                   C.POINTER(RCsrOut)]
        lib.ref_spadd.argtypes = [C.c_int, C.POINTER(OCsrIn), C.c_int, C.POINTER(RCsrOut)]
        lib.ref_mttkrp_dense.argtypes = [C.POINTER(OCsf3), PD, PD, C.c_int64, C.c_int, PD]
        lib.ref_mttkrp_sparse.argtypes = [C.POINTER(OCsf3), C.POINTER(OCsrIn), C.POINTER(OCsrIn),
                                          C.c_int, C.POINTER(RCsrOut)]
        lib.ref_free.argtypes = [C.POINTER(RCsrOut)]
        lib.ref_last_error.restype = C.c_char_p
        _ref = lib
    return _ref


def _np(a):
    if type(a).__module__.startswith("torch"):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(a)


def _csr_in(A, keep):
    pos, idx, vals = _np(A.pos), _np(A.idx), _np(A.vals)
    keep += [pos, idx, vals]
    return OCsrIn(A.nrows, A.ncols, idx.shape[0], pos.ctypes.data_as(P64),
                  idx.ctypes.data_as(P64), vals.ctypes.data_as(PD))


def _csf_in(B, keep):
    arrs = [_np(a) for a in (B.pos1, B.idx1, B.pos2, B.idx2, B.vals)]
    keep += arrs
    v = OCsf3()
    v.dims[0], v.dims[1], v.dims[2] = B.dims
    v.nfibers, v.nnz = arrs[1].shape[0], arrs[3].shape[0]
    v.pos1, v.idx1, v.pos2, v.idx2 = (a.ctypes.data_as(P64) for a in arrs[:4])
    v.vals = arrs[4].ctypes.data_as(PD)
    return v


def _take(res, with_abs):
    n, m = res.nnz, res.nrows + 1
    out = {
        "nrows": res.nrows, "ncols": res.ncols,
        "pos": np.ctypeslib.as_array(res.pos, (m,)).copy(),
        "idx": np.ctypeslib.as_array(res.idx, (n,)).copy() if n else np.zeros(0, np.int64),
        "vals": np.ctypeslib.as_array(res.vals, (n,)).copy() if n else np.zeros(0),
    }
    if with_abs:
        out["abs"] = np.ctypeslib.as_array(res.absv, (n,)).copy() if n else np.zeros(0)
    return out


def threads_default() -> int:
    return os.cpu_count() or 1


# --------------------------------------------------------------------------
# port (C restatement)
def spgemm(A, B, nthreads=1):
    keep = []
    a, b = _csr_in(A, keep), _csr_in(B, keep)
    res = OCsr()
    if port_lib().oracle_spgemm(C.byref(a), C.byref(b), nthreads, C.byref(res)) != 0:
        raise RuntimeError("oracle_spgemm failed")
    out = _take(res, True)
    port_lib().oracle_free(C.byref(res))
    return out


def spadd(ops, nthreads=1):
    keep = []
    arr = (OCsrIn * len(ops))(*[_csr_in(o, keep) for o in ops])
    res = OCsr()
    if port_lib().oracle_spadd(len(ops), arr, nthreads, C.byref(res)) != 0:
        raise RuntimeError("oracle_spadd failed")
    out = _take(res, True)
    port_lib().oracle_free(C.byref(res))
    return out


def ttv(B, c):
    """A(i,j) = sum_k B(i,j,k) c(k) (SPEC Fig. ttv), CSR over B's fibers."""
    keep = []
    b = _csf_in(B, keep)
    cv = np.ascontiguousarray(_np(c), dtype=np.float64)
    res = OCsr()
    if port_lib().oracle_ttv(C.byref(b), cv.ctypes.data_as(PD), C.byref(res)) != 0:
        raise RuntimeError("oracle_ttv failed")
    out = _take(res, True)
    port_lib().oracle_free(C.byref(res))
    return out


def rowdot(Bm, Cm):
    """a(i) = sum_j B(i,j) C(i,j) by two-pointer intersection."""
    keep = []
    b, c = _csr_in(Bm, keep), _csr_in(Cm, keep)
    a = np.empty(Bm.nrows)
    aabs = np.empty(Bm.nrows)
    if port_lib().oracle_rowdot(C.byref(b), C.byref(c), a.ctypes.data_as(PD),
                                aabs.ctypes.data_as(PD)) != 0:
        raise RuntimeError("oracle_rowdot failed")
    return {"vals": a, "abs": aabs}


def spadd_merge(ops):
    """Merge-based SpAdd baseline: ((op0 + op1) + op2) + ... by two-way unions."""
    keep = []
    arr = (OCsrIn * len(ops))(*[_csr_in(o, keep) for o in ops])
    res = OCsr()
    if port_lib().oracle_spadd_merge(len(ops), arr, C.byref(res)) != 0:
        raise RuntimeError("oracle_spadd_merge failed")
    out = _take(res, True)
    port_lib().oracle_free(C.byref(res))
    return out


def mttkrp_dense(B, Cm, Dm, nthreads=1):
    keep = []
    b = _csf_in(B, keep)
    Cn, Dn = _np(Cm), _np(Dm)
    R = Cn.shape[1]
    A = np.empty((B.dims[0], R))
    Aabs = np.empty((B.dims[0], R))
    port_lib().oracle_mttkrp_dense(C.byref(b), Cn.ctypes.data_as(PD), Dn.ctypes.data_as(PD), R,
                                   nthreads, A.ctypes.data_as(PD), Aabs.ctypes.data_as(PD))
    return {"vals": A, "abs": Aabs}


def mttkrp_sparse(B, Cf, Df, nthreads=1):
    keep = []
    b, c, d = _csf_in(B, keep), _csr_in(Cf, keep), _csr_in(Df, keep)
    res = OCsr()
    if port_lib().oracle_mttkrp_sparse(C.byref(b), C.byref(c), C.byref(d), nthreads,
                                       C.byref(res)) != 0:
        raise RuntimeError("oracle_mttkrp_sparse failed")
    out = _take(res, True)
    port_lib().oracle_free(C.byref(res))
    return out


def last_counters() -> dict:
    c = Counters()
    port_lib().oracle_last_counters(C.byref(c))
    return {k: getattr(c, k) for k, _ in Counters._fields_}


# --------------------------------------------------------------------------
# reference (stam::Workspace / TensorBuilder from /root/reference sources)
def _ref_check(rc):
    if rc != 0:
        raise RuntimeError("reference: " + ref_lib().ref_last_error().decode())


def ref_spgemm(A, B, nthreads=1):
    keep = []
    a, b = _csr_in(A, keep), _csr_in(B, keep)
    res = RCsrOut()
    _ref_check(ref_lib().ref_spgemm(C.byref(a), C.byref(b), nthreads, C.byref(res)))
    out = _take(res, False)
    ref_lib().ref_free(C.byref(res))
    return out


def ref_spadd(ops, nthreads=1):
    keep = []
    arr = (OCsrIn * len(ops))(*[_csr_in(o, keep) for o in ops])
    res = RCsrOut()
    _ref_check(ref_lib().ref_spadd(len(ops), arr, nthreads, C.byref(res)))
    out = _take(res, False)
    ref_lib().ref_free(C.byref(res))
    return out


def ref_mttkrp_dense(B, Cm, Dm, nthreads=1):
    keep = []
    b = _csf_in(B, keep)
    Cn, Dn = _np(Cm), _np(Dm)
    R = Cn.shape[1]
    A = np.empty((B.dims[0], R))
    _ref_check(ref_lib().ref_mttkrp_dense(C.byref(b), Cn.ctypes.data_as(PD),
                                          Dn.ctypes.data_as(PD), R, nthreads,
                                          A.ctypes.data_as(PD)))
    return {"vals": A}


def ref_mttkrp_sparse(B, Cf, Df, nthreads=1):
    keep = []
    b, c, d = _csf_in(B, keep), _csr_in(Cf, keep), _csr_in(Df, keep)
    res = RCsrOut()
    _ref_check(ref_lib().ref_mttkrp_sparse(C.byref(b), C.byref(c), C.byref(d), nthreads,
                                           C.byref(res)))
    out = _take(res, False)
    ref_lib().ref_free(C.byref(res))
    return out


# --------------------------------------------------------------------------
def compare_csr(got, ref, rtol=1e-12, exact_values=False) -> dict:
    """Structure bit-exact (pos, idx); values within the scaled criterion
    |x - x_ref| <= rtol * max(|x_ref|, s_ref).  Returns a report;
    raises AssertionError on failure."""
    gp, gi, gv = (_np(got.pos), _np(got.idx), _np(got.vals)) if hasattr(got, "pos") else (
        got["pos"], got["idx"], got["vals"])
    assert gp.shape == ref["pos"].shape and np.array_equal(gp, ref["pos"]), "pos differs"
    assert gi.shape == ref["idx"].shape and np.array_equal(gi, ref["idx"]), "idx differs"
    rv = ref["vals"]
    if exact_values:
        same = np.array_equal(gv.view(np.int64), rv.view(np.int64))
        assert same, f"values not bit-identical ({int(np.sum(gv != rv))} differ)"
    scale = np.maximum(np.abs(rv), ref.get("abs", np.abs(rv)))
    err = np.abs(gv - rv)
    bad = err > rtol * scale
    assert not np.any(bad), f"{int(bad.sum())} values outside tolerance, max {err.max():.3e}"
    nz = np.abs(rv) > 0
    rel = np.where(nz, err / np.where(nz, np.abs(rv), 1), 0)
    return {"nnz": int(rv.shape[0]), "max_abs_err": float(err.max()) if err.size else 0.0,
            "max_rel_err": float(rel.max()) if rel.size else 0.0,
            "bit_identical": bool(np.array_equal(gv.view(np.int64), rv.view(np.int64)))}
