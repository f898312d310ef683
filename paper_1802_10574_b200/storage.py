"""Python mirror of the reference storage types at the hot path's boundary.

``CSR``, ``CSF3`` and ``Dense`` are the three ``stam::TensorStorage`` shapes the
kernels consume and produce (``include/stam/storage.h:17-72``):

* ``CSR``  — format ``csr()`` = {dense, compressed} (``src/format.cpp:83``):
  ``level(1).pos`` int64[nrows+1], ``level(1).idx`` int64[nnz], ``vals`` fp64[nnz].
* ``CSF3`` — format ``csf(3)`` = {dense, compressed, compressed}
  (``src/format.cpp:91-95``): pos1/idx1 for the j level, pos2/idx2 for k.
* ``Dense`` — ``denseFormat(2)``, row-major (``storage.cpp:69-70``).

Arrays are numpy (host) or torch tensors (host or CUDA).  ``validate`` restates
``TensorStorage::validate`` (``src/storage.cpp:103-147``) and raises the same
``ErrorCode`` family (``Internal`` for broken invariants).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Any

import numpy as np

from . import _native as N


def _is_torch(a: Any) -> bool:
    return type(a).__module__.startswith("torch")


def _on_device(a: Any) -> bool:
    return _is_torch(a) and a.is_cuda


def _ptr(a: Any) -> int:
    if a is None:
        return 0
    if _is_torch(a):
        if not a.is_contiguous():
            raise N.StamError(8, "arrays must be contiguous")
        return a.data_ptr()
    if not a.flags["C_CONTIGUOUS"]:
        raise N.StamError(8, "arrays must be contiguous")
    return a.ctypes.data


def _check_dtype(a: Any, want: str, what: str) -> None:
    name = str(a.dtype).replace("torch.", "")
    if name != want:
        raise N.StamError(8, f"{what} must be {want}, got {name}")


def _np(a: Any) -> np.ndarray:
    if _is_torch(a):
        return a.detach().cpu().numpy()
    return np.asarray(a)


def _mem(arrays) -> int:
    kinds = {_on_device(a) for a in arrays if a is not None}
    if len(kinds) > 1:
        raise N.StamError(8, "arrays of one tensor must all be on the host or all on the device")
    return N.STAM_MEM_DEVICE if kinds == {True} else N.STAM_MEM_HOST


def _to(a: Any, device: str):
    import torch

    if device == "cpu":
        return _np(a)
    t = a if _is_torch(a) else torch.from_numpy(np.ascontiguousarray(a))
    return t.to(device)


@dataclass
class CSR:
    nrows: int
    ncols: int
    pos: Any
    idx: Any
    vals: Any

    @property
    def nnz(self) -> int:
        return int(self.idx.shape[0])

    @property
    def dimensions(self) -> list[int]:
        return [self.nrows, self.ncols]

    def view(self) -> N.CsrView:
        _check_dtype(self.pos, "int64", "pos")
        _check_dtype(self.idx, "int64", "idx")
        _check_dtype(self.vals, "float64", "vals")
        if self.pos.shape[0] != self.nrows + 1:
            raise N.StamError(21, "pos array length != rows + 1")
        if self.vals.shape[0] != self.idx.shape[0]:
            raise N.StamError(21, "value array length != idx length")
        return N.CsrView(self.nrows, self.ncols, self.nnz, _ptr(self.pos), _ptr(self.idx),
                         _ptr(self.vals), _mem([self.pos, self.idx, self.vals]), 0)

    def to(self, device: str) -> "CSR":
        return CSR(self.nrows, self.ncols, _to(self.pos, device), _to(self.idx, device),
                   _to(self.vals, device))

    def numpy(self) -> "CSR":
        return self.to("cpu")

    def validate(self) -> None:
        """TensorStorage::validate for csr() (storage.cpp:103-147)."""
        pos, idx, vals = _np(self.pos), _np(self.idx), _np(self.vals)
        if self.nrows <= 0 or self.ncols <= 0:
            raise N.StamError(3, "dimensions must be positive")
        if pos.shape[0] != self.nrows + 1:
            raise N.StamError(21, "pos array length != parent positions + 1")
        if pos[0] != 0:
            raise N.StamError(21, "pos[0] != 0")
        if np.any(np.diff(pos) < 0):
            raise N.StamError(21, "pos array is not nondecreasing")
        if pos[-1] != idx.shape[0]:
            raise N.StamError(21, "pos[last] != length(idx)")
        if idx.size and (idx.min() < 0 or idx.max() >= self.ncols):
            raise N.StamError(21, "idx entry out of range")
        if idx.size > 1:
            inc = np.diff(idx) > 0
            row_start = np.zeros(idx.shape[0], dtype=bool)
            starts = pos[:-1][pos[:-1] < idx.shape[0]]
            row_start[starts] = True
            if np.any(~inc & ~row_start[1:]):
                raise N.StamError(21, "coordinates not strictly increasing in ordered level")
        if vals.shape[0] != idx.shape[0]:
            raise N.StamError(21, "value array length != last level positions")

    def to_dense(self) -> np.ndarray:
        pos, idx, vals = _np(self.pos), _np(self.idx), _np(self.vals)
        out = np.zeros((self.nrows, self.ncols))
        rows = np.repeat(np.arange(self.nrows), np.diff(pos))
        np.add.at(out, (rows, idx), vals)
        return out

    @staticmethod
    def from_dense(m: np.ndarray) -> "CSR":
        m = np.asarray(m, dtype=np.float64)
        rows, cols = np.nonzero(m)
        pos = np.zeros(m.shape[0] + 1, dtype=np.int64)
        np.add.at(pos, rows + 1, 1)
        pos = np.cumsum(pos).astype(np.int64)
        return CSR(m.shape[0], m.shape[1], pos, cols.astype(np.int64), m[rows, cols].copy())


@dataclass
class CSF3:
    dims: tuple[int, int, int]
    pos1: Any
    idx1: Any
    pos2: Any
    idx2: Any
    vals: Any

    @property
    def nnz(self) -> int:
        return int(self.idx2.shape[0])

    @property
    def nfibers(self) -> int:
        return int(self.idx1.shape[0])

    def view(self) -> N.Csf3View:
        for a, w in ((self.pos1, "pos1"), (self.idx1, "idx1"), (self.pos2, "pos2"),
                     (self.idx2, "idx2")):
            _check_dtype(a, "int64", w)
        _check_dtype(self.vals, "float64", "vals")
        if self.pos1.shape[0] != self.dims[0] + 1 or self.pos2.shape[0] != self.nfibers + 1:
            raise N.StamError(21, "pos array length != parent positions + 1")
        v = N.Csf3View()
        v.dims[0], v.dims[1], v.dims[2] = self.dims
        v.nfibers, v.nnz = self.nfibers, self.nnz
        v.pos1, v.idx1, v.pos2 = _ptr(self.pos1), _ptr(self.idx1), _ptr(self.pos2)
        v.idx2, v.vals = _ptr(self.idx2), _ptr(self.vals)
        v.mem = _mem([self.pos1, self.idx1, self.pos2, self.idx2, self.vals])
        return v

    def to(self, device: str) -> "CSF3":
        return CSF3(tuple(self.dims), *(_to(a, device) for a in
                                        (self.pos1, self.idx1, self.pos2, self.idx2, self.vals)))

    def numpy(self) -> "CSF3":
        return self.to("cpu")

    def validate(self) -> None:
        pos1, idx1, pos2, idx2, vals = map(_np, (self.pos1, self.idx1, self.pos2, self.idx2,
                                                 self.vals))
        I, J, K = self.dims
        for pos, parents, child, dim in ((pos1, I, idx1, J), (pos2, idx1.shape[0], idx2, K)):
            if pos.shape[0] != parents + 1 or pos[0] != 0 or pos[-1] != child.shape[0]:
                raise N.StamError(21, "pos array inconsistent")
            if np.any(np.diff(pos) < 0):
                raise N.StamError(21, "pos array is not nondecreasing")
            if child.size and (child.min() < 0 or child.max() >= dim):
                raise N.StamError(21, "idx entry out of range")
            if child.size > 1:
                inc = np.diff(child) > 0
                start = np.zeros(child.shape[0], dtype=bool)
                start[pos[:-1][pos[:-1] < child.shape[0]]] = True
                if np.any(~inc & ~start[1:]):
                    raise N.StamError(21, "coordinates not strictly increasing")
        if vals.shape[0] != idx2.shape[0]:
            raise N.StamError(21, "value array length != last level positions")

    def to_dense(self) -> np.ndarray:
        pos1, idx1, pos2, idx2, vals = map(_np, (self.pos1, self.idx1, self.pos2, self.idx2,
                                                 self.vals))
        out = np.zeros(self.dims)
        fib_i = np.repeat(np.arange(self.dims[0]), np.diff(pos1))
        nz_f = np.repeat(np.arange(idx1.shape[0]), np.diff(pos2))
        out[fib_i[nz_f], idx1[nz_f], idx2] = vals
        return out

    @staticmethod
    def from_dense(t: np.ndarray) -> "CSF3":
        t = np.asarray(t, dtype=np.float64)
        I, J, K = t.shape
        ii, jj, kk = np.nonzero(t)  # lexicographic order
        fib_key = ii * J + jj
        new_fib = np.ones(ii.shape[0], dtype=bool)
        new_fib[1:] = fib_key[1:] != fib_key[:-1]
        fib_i = ii[new_fib]
        idx1 = jj[new_fib].astype(np.int64)
        pos1 = np.zeros(I + 1, dtype=np.int64)
        np.add.at(pos1, fib_i + 1, 1)
        pos1 = np.cumsum(pos1).astype(np.int64)
        starts = np.nonzero(new_fib)[0]
        pos2 = np.append(starts, ii.shape[0]).astype(np.int64)
        return CSF3((I, J, K), pos1, idx1, pos2, kk.astype(np.int64), t[ii, jj, kk].copy())


@dataclass
class Dense:
    vals: Any  # 2-D, row-major

    @property
    def nrows(self) -> int:
        return int(self.vals.shape[0])

    @property
    def ncols(self) -> int:
        return int(self.vals.shape[1])

    def view(self) -> N.DenseView:
        _check_dtype(self.vals, "float64", "vals")
        return N.DenseView(self.nrows, self.ncols, _ptr(self.vals), _mem([self.vals]), 0)

    def to(self, device: str) -> "Dense":
        return Dense(_to(self.vals, device))

    def numpy(self) -> np.ndarray:
        return _np(self.vals)
