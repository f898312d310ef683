"""Exchange formats, mirroring ``include/stam/io.h``:
Matrix Market coordinate files and FROSTT ``.tns`` files to and from the
``CSR`` / ``CSF3`` containers.  Duplicates are summed in file order, Matrix
Market symmetric / skew-symmetric files are expanded to general, pattern
entries get 1.0, and values are written with 17 significant digits so
``load(store(x)) == x``.  Errors raise ``StamError`` with the reference codes
(``Io`` for malformed input, naming the line; ``OutOfRange`` for coordinates
outside the matrix or 0-based files)."""
from __future__ import annotations

from pathlib import Path
from typing import Optional, Sequence, Union

import numpy as np

from ._native import StamError
from .storage import CSF3, CSR

_IO, _OUT_OF_RANGE, _DIM = 20, 5, 3


def _fail(code: int, msg: str):
    raise StamError(code, msg)


def _parse_rows(lines, first_line_no: int, path: str, ncols_min: int, ncols_max: int):
    """Whitespace-separated numeric rows -> float64 matrix (with line checks)."""
    out = []
    for k, ln in enumerate(lines):
        parts = ln.split()
        if not (ncols_min <= len(parts) <= ncols_max):
            _fail(_IO, f"{path}:{first_line_no + k}: malformed entry")
        try:
            out.append([float(x) for x in parts])
        except ValueError:
            _fail(_IO, f"{path}:{first_line_no + k}: malformed entry")
    return out


def _coo_sum(coords: np.ndarray, vals: np.ndarray):
    """Stable sort by coordinates; duplicates summed sequentially in file order."""
    order = np.lexsort(coords.T[::-1])
    c, v = coords[order], vals[order]
    if c.shape[0] == 0:
        return c, v
    new = np.ones(c.shape[0], dtype=bool)
    new[1:] = np.any(c[1:] != c[:-1], axis=1)
    starts = np.flatnonzero(new)
    uv = v[starts].copy()
    ends = np.append(starts[1:], c.shape[0])
    for g in np.flatnonzero(ends - starts > 1):  # rare: sequential sum in file order
        acc = v[starts[g]]
        for t in range(starts[g] + 1, ends[g]):
            acc = acc + v[t]
        uv[g] = acc
    return c[starts], uv


def _csr_from_coo(rows: int, cols: int, c: np.ndarray, v: np.ndarray) -> CSR:
    pos = np.zeros(rows + 1, dtype=np.int64)
    np.add.at(pos, c[:, 0] + 1, 1)
    np.cumsum(pos, out=pos)
    return CSR(rows, cols, pos, c[:, 1].astype(np.int64).copy(), v.astype(np.float64))


def _csf3_from_coo(dims, c: np.ndarray, v: np.ndarray) -> CSF3:
    n = c.shape[0]
    newf = np.ones(n, dtype=bool)
    if n:
        newf[1:] = np.any(c[1:, :2] != c[:-1, :2], axis=1)
    fstart = np.flatnonzero(newf)
    pos2 = np.append(fstart, n).astype(np.int64)
    idx1 = c[fstart, 1].astype(np.int64)
    pos1 = np.zeros(dims[0] + 1, dtype=np.int64)
    np.add.at(pos1, c[fstart, 0] + 1, 1)
    np.cumsum(pos1, out=pos1)
    return CSF3(tuple(int(d) for d in dims), pos1, idx1, pos2, c[:, 2].astype(np.int64).copy(),
                v.astype(np.float64))


def load_matrix_market(path: Union[str, Path]) -> CSR:
    path = str(path)
    try:
        text = Path(path).read_text().splitlines()
    except OSError as e:
        _fail(_IO, f"cannot open {path}: {e}")
    if not text:
        _fail(_IO, f"{path}:1: empty file")
    h = text[0].lower().split()
    if len(h) < 5 or h[0] != "%%matrixmarket" or h[1] != "matrix":
        _fail(_IO, f"{path}:1: not a Matrix Market matrix header")
    if h[2] != "coordinate":
        _fail(_IO, f"{path}:1: only the coordinate format is supported")
    field, sym = h[3], h[4]
    if field not in ("real", "integer", "double", "pattern"):
        _fail(_IO, f"{path}:1: unsupported field '{field}'")
    if sym not in ("general", "symmetric", "skew-symmetric"):
        _fail(_IO, f"{path}:1: unsupported symmetry '{sym}'")
    k = 1
    while k < len(text) and (text[k].startswith("%") or not text[k].strip()):
        k += 1
    if k >= len(text):
        _fail(_IO, f"{path}:{k}: missing size line")
    try:
        rows, cols, nnz = (int(x) for x in text[k].split())
    except ValueError:
        _fail(_IO, f"{path}:{k + 1}: malformed size line")
    body = [(n + k + 2, ln) for n, ln in enumerate(text[k + 1:])
            if ln.strip() and not ln.startswith("%")]
    if len(body) < nnz:
        _fail(_IO, f"{path}: fewer entries than the size line announces")
    body = body[:nnz]
    want = 2 if field == "pattern" else 3
    data = np.zeros((nnz, 3))
    for t, (no, ln) in enumerate(body):
        parts = ln.split()
        if len(parts) != want:
            _fail(_IO, f"{path}:{no}: malformed entry")
        try:
            data[t, 0], data[t, 1] = int(parts[0]), int(parts[1])
            data[t, 2] = 1.0 if field == "pattern" else float(parts[2])
        except ValueError:
            _fail(_IO, f"{path}:{no}: malformed entry")
    ij = data[:, :2].astype(np.int64)
    if nnz and (ij.min() < 1 or ij[:, 0].max() > rows or ij[:, 1].max() > cols):
        _fail(_OUT_OF_RANGE, f"{path}: coordinate out of range")
    ij -= 1
    v = data[:, 2]
    if sym != "general":
        off = ij[:, 0] != ij[:, 1]
        # interleave each off-diagonal entry with its mirror (file order)
        mirror = ij[off][:, ::-1]
        mv = -v[off] if sym == "skew-symmetric" else v[off]
        allc = np.empty((nnz + int(off.sum()), 2), dtype=np.int64)
        allv = np.empty(allc.shape[0])
        slot = np.arange(nnz) + np.concatenate([[0], np.cumsum(off)[:-1]])
        allc[slot], allv[slot] = ij, v
        ms = slot[off] + 1
        allc[ms], allv[ms] = mirror, mv
        ij, v = allc, allv
    c, uv = _coo_sum(ij, v)
    return _csr_from_coo(rows, cols, c, uv)


def load_tns(path: Union[str, Path], dims: Optional[Sequence[int]] = None):
    """Order 3 -> CSF3, order 2 -> CSR."""
    path = str(path)
    try:
        text = Path(path).read_text().splitlines()
    except OSError as e:
        _fail(_IO, f"cannot open {path}: {e}")
    body = [(n + 1, ln) for n, ln in enumerate(text) if ln.strip() and not ln.lstrip().startswith("#")]
    if not body:
        _fail(_IO, f"{path}: no entries (the order of an empty .tns file is unknown)")
    order = len(body[0][1].split()) - 1
    if order < 1:
        _fail(_IO, f"{path}:{body[0][0]}: malformed entry")
    coords = np.zeros((len(body), order), dtype=np.int64)
    vals = np.zeros(len(body))
    for t, (no, ln) in enumerate(body):
        parts = ln.split()
        if len(parts) != order + 1:
            _fail(_IO, f"{path}:{no}: malformed entry")
        try:
            coords[t] = [int(x) for x in parts[:order]]
            vals[t] = float(parts[order])
        except ValueError:
            _fail(_IO, f"{path}:{no}: malformed entry")
    if coords.min() < 1:
        _fail(_OUT_OF_RANGE, f"{path}: coordinates are 1-based")
    maxc = coords.max(axis=0)
    d = list(maxc) if dims is None else list(dims)
    if len(d) != order:
        _fail(_DIM, "load_tns: dims order mismatch")
    if np.any(maxc > np.asarray(d)):
        _fail(_OUT_OF_RANGE, "load_tns: coordinate beyond the given dimension")
    c, uv = _coo_sum(coords - 1, vals)
    if order == 2:
        return _csr_from_coo(int(d[0]), int(d[1]), c, uv)
    if order == 3:
        return _csf3_from_coo(d, c, uv)
    _fail(_DIM, "load_tns: only orders 2 and 3 have containers in this package")


def _entries(obj):
    if isinstance(obj, CSR):
        pos = np.asarray(obj.pos)
        rows = np.repeat(np.arange(obj.nrows), np.diff(pos))
        return np.stack([rows, np.asarray(obj.idx)], axis=1), np.asarray(obj.vals), (obj.nrows, obj.ncols)
    if isinstance(obj, CSF3):
        pos1, pos2 = np.asarray(obj.pos1), np.asarray(obj.pos2)
        fi = np.repeat(np.arange(obj.dims[0]), np.diff(pos1))
        i = np.repeat(fi, np.diff(pos2))
        j = np.repeat(np.asarray(obj.idx1), np.diff(pos2))
        return np.stack([i, j, np.asarray(obj.idx2)], axis=1), np.asarray(obj.vals), obj.dims
    raise TypeError("store: CSR or CSF3 expected")


def store(path: Union[str, Path], obj) -> None:
    """.mtx (CSR) as 'matrix coordinate real general', anything else as .tns."""
    path = str(path)
    c, v, dims = _entries(obj)
    with open(path, "w") as f:
        if path.endswith(".mtx"):
            if len(dims) != 2:
                _fail(_DIM, "store: .mtx needs order 2")
            f.write("%%MatrixMarket matrix coordinate real general\n")
            f.write(f"{dims[0]} {dims[1]} {len(v)}\n")
        for row, val in zip(c + 1, v):
            f.write(" ".join(str(int(x)) for x in row) + f" {float(val):.17g}\n")
