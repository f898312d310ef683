"""Seeded synthetic inputs with the shapes of BASELINE.json's five configs.

The real SuiteSparse / FROSTT (NELL-2) inputs are not available offline;
these generators stand in for them with the stated shapes, sizes and value
distributions:

1. SpGEMM 10k x 10k, 20 distinct sorted columns per row, values U[-1,1).
2. SpAdd 3 x 200k x 200k, 50 per row, values U[-1,1).
3. SpGEMM A·A, 1M x 1M, row lengths P(L) ∝ (L + 1.7764)^-2 on [1, 5000]
   (exponent 2, mean 16.0: the literal "Zipf 2.0, mean 16" is inconsistent,
   SURVEY P2), i.i.d. per row (= shuffled), values U[-1,1).
4. MTTKRP dense: CSF 12,092 x 9,184 x 28,818, 76,879,419 nnz, i-slice sizes
   rank-size r^-1.5 scaled to the total (largest remainder, min 1) assigned by a
   seeded shuffle, (j,k) distinct uniform per slice, values U[0,1); C, D dense
   rank 32, values U[-1,1).
5. MTTKRP sparse: CSF 500k^3 with 200M nnz, i uniform per nonzero, (j,k)
   distinct uniform per slice, values U[0,1); C, D CSR 500k x 256 with 8
   distinct sorted columns per row, values U[-1,1).

``scale`` shrinks a config (rows / slices / nnz) for parity tests while keeping
its distributions.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .storage import CSF3, CSR, Dense

_LIB = Path(__file__).resolve().parent / "_lib" / "libstamgen.so"
_gen = None

P64 = C.POINTER(C.c_int64)
PD = C.POINTER(C.c_double)


def _lib():
    global _gen
    if _gen is None:
        if not _LIB.exists():
            raise ImportError(f"{_LIB} missing; run __graft_entry__.build()")
        g = C.CDLL(str(_LIB))
        g.gen_powerlaw_pos.restype = C.c_int64
        g.gen_powerlaw_pos.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_int64, C.c_int64,
                                       C.c_uint64, P64]
        g.gen_csr_fill.restype = C.c_int
        g.gen_csr_fill.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_double, C.c_double, P64,
                                   P64, PD, C.c_int]
        g.gen_uniform_slice_counts.restype = C.c_int
        g.gen_uniform_slice_counts.argtypes = [C.c_int64, C.c_int64, C.c_uint64, P64, C.c_int]
        g.gen_csf3_plan.restype = C.c_int
        g.gen_csf3_plan.argtypes = [C.c_int64, C.c_int64, C.c_int64, P64, C.c_uint64, P64, C.c_int]
        g.gen_csf3_fill.restype = C.c_int
        g.gen_csf3_fill.argtypes = [C.c_int64, C.c_int64, C.c_int64, P64, C.c_uint64, P64, P64, P64,
                                    P64, P64, PD, C.c_double, C.c_double, C.c_int]
        g.gen_dense.restype = C.c_int
        g.gen_dense.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_double, C.c_double, PD,
                                C.c_int]
        _gen = g
    return _gen


def _threads() -> int:
    return max(1, min(64, os.cpu_count() or 1))


def _p64(a):
    return a.ctypes.data_as(P64)


def _pd(a):
    return a.ctypes.data_as(PD)


def csr_from_lengths(nrows: int, ncols: int, pos: np.ndarray, seed: int, lo=-1.0, hi=1.0) -> CSR:
    nnz = int(pos[-1])
    idx = np.empty(nnz, dtype=np.int64)
    vals = np.empty(nnz, dtype=np.float64)
    rc = _lib().gen_csr_fill(nrows, ncols, seed, lo, hi, _p64(pos), _p64(idx), _pd(vals),
                             _threads())
    if rc != 0:
        raise ValueError("row longer than the number of columns")
    return CSR(nrows, ncols, pos, idx, vals)


def csr_fixed(nrows: int, ncols: int, per_row: int, seed: int, lo=-1.0, hi=1.0) -> CSR:
    pos = (np.arange(nrows + 1, dtype=np.int64) * per_row).astype(np.int64)
    return csr_from_lengths(nrows, ncols, pos, seed, lo, hi)


def csr_powerlaw(nrows: int, ncols: int, seed: int, a=2.0, q=1.7764, lmin=1, lmax=5000,
                 lo=-1.0, hi=1.0) -> CSR:
    lmax = min(lmax, ncols)
    pos = np.empty(nrows + 1, dtype=np.int64)
    _lib().gen_powerlaw_pos(nrows, a, q, lmin, lmax, seed, _p64(pos))
    return csr_from_lengths(nrows, ncols, pos, seed, lo, hi)


def dense(nrows: int, ncols: int, seed: int, lo=-1.0, hi=1.0) -> Dense:
    out = np.empty((nrows, ncols), dtype=np.float64)
    _lib().gen_dense(nrows, ncols, seed, lo, hi, _pd(out), _threads())
    return Dense(out)


def slice_sizes_ranksize(nslices: int, nnz: int, alpha: float, seed: int,
                         cap: int | None = None) -> np.ndarray:
    """Rank-size law s_r ∝ r^-alpha scaled to `nnz` (largest remainder, min 1),
    assigned to slices by a seeded shuffle."""
    r = np.arange(1, nslices + 1, dtype=np.float64)
    w = r ** -alpha
    target = w / w.sum() * (nnz - nslices)  # reserve the minimum of 1 per slice
    base = np.floor(target).astype(np.int64)
    rem = (nnz - nslices) - int(base.sum())
    order = np.argsort(-(target - base), kind="stable")
    base[order[:rem]] += 1
    sizes = base + 1
    if cap is not None and sizes.max() > cap:
        raise ValueError("slice larger than J*K")
    perm = np.random.Generator(np.random.PCG64(seed)).permutation(nslices)
    out = np.empty(nslices, dtype=np.int64)
    out[perm] = sizes
    return out


def slice_sizes_uniform(nslices: int, nnz: int, seed: int) -> np.ndarray:
    counts = np.empty(nslices, dtype=np.int64)
    _lib().gen_uniform_slice_counts(nslices, nnz, seed, _p64(counts), _threads())
    return counts


def csf3(dims, slice_nnz: np.ndarray, seed: int, lo=0.0, hi=1.0) -> CSF3:
    I, J, K = (int(d) for d in dims)
    slice_nnz = np.ascontiguousarray(slice_nnz, dtype=np.int64)
    fibers = np.empty(I, dtype=np.int64)
    if _lib().gen_csf3_plan(I, J, K, _p64(slice_nnz), seed, _p64(fibers), _threads()) != 0:
        raise ValueError("slice larger than J*K")
    pos1 = np.zeros(I + 1, dtype=np.int64)
    np.cumsum(fibers, out=pos1[1:])
    nz_off = np.zeros(I + 1, dtype=np.int64)
    np.cumsum(slice_nnz, out=nz_off[1:])
    nf, nnz = int(pos1[-1]), int(nz_off[-1])
    idx1 = np.empty(nf, dtype=np.int64)
    pos2 = np.empty(nf + 1, dtype=np.int64)
    idx2 = np.empty(nnz, dtype=np.int64)
    vals = np.empty(nnz, dtype=np.float64)
    _lib().gen_csf3_fill(I, J, K, _p64(slice_nnz), seed, _p64(pos1), _p64(nz_off), _p64(idx1),
                         _p64(pos2), _p64(idx2), _pd(vals), lo, hi, _threads())
    return CSF3((I, J, K), pos1, idx1, pos2, idx2, vals)


# ---------------------------------------------------------------------------
# BASELINE configs
# ---------------------------------------------------------------------------
CONFIG_NAMES = {
    1: "spgemm_10k_20perrow",
    2: "spadd3_200k_50perrow",
    3: "spgemm_AxA_1M_powerlaw",
    4: "mttkrp_dense_nell2shape_R32",
    5: "mttkrp_sparse_500k3_200M_R256",
}

KIND = {1: "spgemm", 2: "spadd", 3: "spgemm", 4: "mttkrp_dense", 5: "mttkrp_sparse"}

SEEDS = {1: (101, 102), 2: (201, 202, 203), 3: (301,), 4: (401, 402, 403, 404),
         5: (501, 502, 503, 504)}


def make_config(cid: int, scale: float = 1.0, shard: int = 0) -> dict:
    """Inputs for BASELINE config `cid` (1..5).  `scale` < 1 shrinks rows /
    slices / nnz proportionally; `shard` offsets every seed (independent
    per-rank inputs for weak scaling)."""
    s = [x + 1000003 * shard for x in SEEDS[cid]]
    if cid == 1:
        n = max(32, int(10_000 * scale))
        A = csr_fixed(n, n, min(20, n), s[0])
        B = csr_fixed(n, n, min(20, n), s[1])
        return {"kind": "spgemm", "A": A, "B": B}
    if cid == 2:
        n = max(32, int(200_000 * scale))
        ops = [csr_fixed(n, n, min(50, n), x) for x in s]
        return {"kind": "spadd", "ops": ops}
    if cid == 3:
        n = max(64, int(1_000_000 * scale))
        A = csr_powerlaw(n, n, s[0], lmax=min(5000, n))
        return {"kind": "spgemm", "A": A, "B": A}
    if cid == 4:
        I, J, K = 12_092, 9_184, 28_818
        nnz = 76_879_419
        if scale < 1.0:
            I = max(16, int(I * scale))
            J = max(16, int(J * scale ** 0.5))
            K = max(16, int(K * scale ** 0.5))
            nnz = max(I, int(nnz * scale * scale))
        sizes = slice_sizes_ranksize(I, nnz, 1.5, s[3], cap=J * K)
        B = csf3((I, J, K), sizes, s[0], 0.0, 1.0)
        R = 32
        return {"kind": "mttkrp_dense", "B": B, "C": dense(J, R, s[1]), "D": dense(K, R, s[2])}
    if cid == 5:
        I = J = K = 500_000
        nnz = 200_000_000
        if scale < 1.0:
            I = J = K = max(64, int(500_000 * scale))
            nnz = max(I, int(nnz * scale))
        sizes = slice_sizes_uniform(I, nnz, s[3])
        B = csf3((I, J, K), sizes, s[0], 0.0, 1.0)
        R = 256
        per = 8
        Cf = csr_fixed(J, R, per, s[1])
        Df = csr_fixed(K, R, per, s[2])
        return {"kind": "mttkrp_sparse", "B": B, "C": Cf, "D": Df}
    raise ValueError(f"unknown config {cid}")
