"""Multi-GPU sharding of the hot path: one process per GPU,
``torch.distributed`` (NCCL over NVLink/NVSwitch on GPUs, gloo on CPU for tests).

Rank 0 holds the problem (it generated or loaded it).  It computes the
partition from host metadata (pos arrays only), ships every rank its own block
once (point-to-point sends: a scatter), and broadcasts the operand every rank
reads in full once.  Everything a rank receives stays resident on its device
(``device="cuda"``; on ``"cpu"`` the same code runs over gloo for the tests).

* SpGEMM  — contiguous row blocks of A balanced by the prefix of per-row
  products (sum over A(i,:) of nnz(B_k)); B is broadcast once.  When B *is* A
  (config 3's A·A) only A is broadcast and each rank's row block is a view of
  the broadcast copy.
* SpAdd   — contiguous row blocks balanced by operand nnz; nothing broadcast.
* MTTKRP  — factors broadcast once.  Dense result: contiguous fiber blocks
  balanced by nnz (cut inside slices: config 4's heaviest slice holds 38.5 %
  of the nonzeros); the only data-path exchange is one all-gather of each
  rank's first partial row (the <= N-1 cut slices), added by the slice's
  owner in rank order (deterministic).  Sparse result: nnz-balanced i-slice
  blocks (slice-aligned; a result row is one compacted workspace).

Outputs stay row-sharded; ``concat_csr`` reassembles a global CSR when asked
(pos arrays offset by the preceding shards' nnz).

``compute`` callables are injected so the same orchestration runs the CUDA
kernels on GPUs and (in tests) any CPU callable on gloo.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np

from .storage import CSF3, CSR


def _np(a):
    if type(a).__module__.startswith("torch"):
        return a.detach().cpu().numpy()
    return np.asarray(a)


def balanced_bounds(weights: np.ndarray, nparts: int) -> np.ndarray:
    """Contiguous partition of len(weights) items into nparts blocks with
    nearly equal total weight: bounds[p]..bounds[p+1] is block p."""
    w = np.asarray(weights, dtype=np.float64)
    n = w.shape[0]
    if nparts <= 1 or n == 0:
        return np.array([0, n], dtype=np.int64)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    if total <= 0:
        return np.linspace(0, n, nparts + 1).round().astype(np.int64)
    targets = total * np.arange(1, nparts) / nparts
    inner = np.searchsorted(cum, targets, side="left")
    bounds = np.concatenate([[0], np.clip(inner, 0, n), [n]]).astype(np.int64)
    return np.maximum.accumulate(bounds)


def spgemm_row_weights(A: CSR, B: CSR) -> np.ndarray:
    """Products per row of A·B (the binning key and the balance weight)."""
    blen = np.diff(_np(B.pos))
    prod = blen[_np(A.idx)]
    rows = np.repeat(np.arange(A.nrows), np.diff(_np(A.pos)))
    return np.bincount(rows, weights=prod, minlength=A.nrows)


def csr_rows(A: CSR, r0: int, r1: int) -> CSR:
    pos = _np(A.pos)
    a, b = int(pos[r0]), int(pos[r1])
    return CSR(r1 - r0, A.ncols, (pos[r0:r1 + 1] - a).astype(np.int64), _np(A.idx)[a:b],
               _np(A.vals)[a:b])


def csf_slices(B: CSF3, i0: int, i1: int) -> CSF3:
    pos1, pos2 = _np(B.pos1), _np(B.pos2)
    f0, f1 = int(pos1[i0]), int(pos1[i1])
    z0, z1 = int(pos2[f0]), int(pos2[f1])
    return CSF3((i1 - i0, B.dims[1], B.dims[2]), (pos1[i0:i1 + 1] - f0).astype(np.int64),
                _np(B.idx1)[f0:f1], (pos2[f0:f1 + 1] - z0).astype(np.int64),
                _np(B.idx2)[z0:z1], _np(B.vals)[z0:z1])


def concat_csr(parts: Sequence[CSR]) -> CSR:
    """Row-shard results -> one global CSR."""
    poss, idxs, vals = [np.zeros(1, dtype=np.int64)], [], []
    off = 0
    for p in parts:
        pp = _np(p.pos)
        poss.append(pp[1:] + off)
        off += int(pp[-1])
        idxs.append(_np(p.idx))
        vals.append(_np(p.vals))
    return CSR(sum(p.nrows for p in parts), parts[0].ncols, np.concatenate(poss),
               np.concatenate(idxs) if idxs else np.zeros(0, np.int64),
               np.concatenate(vals) if vals else np.zeros(0))


def fiber_bounds(B: CSF3, nparts: int) -> np.ndarray:
    """Contiguous fiber ranges with nearly equal nnz (cut at fiber, not slice,
    boundaries: config 4's largest i-slice holds 38.5 % of the nonzeros, which
    slice-aligned blocks would leave on one GPU)."""
    return balanced_bounds(np.diff(_np(B.pos2)), nparts)


def csf_fibers(B: CSF3, f0: int, f1: int):
    """Fibers [f0, f1) as a CSF over the slices they touch: returns (s0, sub)
    with sub's slice 0 = B's slice s0 (possibly a partial slice at either end)."""
    pos1, pos2 = _np(B.pos1), _np(B.pos2)
    if f1 <= f0:
        return 0, CSF3((0, B.dims[1], B.dims[2]), np.zeros(1, np.int64), np.zeros(0, np.int64),
                       np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    s0 = int(np.searchsorted(pos1, f0, side="right") - 1)
    s1 = int(np.searchsorted(pos1, f1 - 1, side="right"))  # one past the last touched slice
    p1 = np.clip(pos1[s0:s1 + 1], f0, f1) - f0
    z0, z1 = int(pos2[f0]), int(pos2[f1])
    return s0, CSF3((s1 - s0, B.dims[1], B.dims[2]), p1.astype(np.int64), _np(B.idx1)[f0:f1],
                    (pos2[f0:f1 + 1] - z0).astype(np.int64), _np(B.idx2)[z0:z1],
                    _np(B.vals)[z0:z1])


# ---------------------------------------------------------------------------
# transport (torch.distributed): broadcast once, scatter blocks point-to-point
# ---------------------------------------------------------------------------
def _dist():
    import torch.distributed as dist

    return dist


def _torch_dtype(np_dtype):
    import torch

    return {np.dtype(np.int64): torch.int64, np.dtype(np.float64): torch.float64}[np.dtype(np_dtype)]


def _upload(a, device):
    """Host (numpy / torch) or device array -> contiguous tensor on `device`."""
    import torch

    t = a if type(a).__module__.startswith("torch") else torch.from_numpy(np.ascontiguousarray(a))
    return t.to(device).contiguous()


def _out(t, device):
    return t if device != "cpu" else t.numpy()


def broadcast_arrays(arrays, dtypes, src: int, device: str):
    """Arrays held by `src` -> every rank (one broadcast per array)."""
    import torch

    dist = _dist()
    rank = dist.get_rank()
    n = len(dtypes)
    meta = torch.zeros(n, dtype=torch.int64, device=device)
    if rank == src:
        meta[:] = torch.tensor([int(np.asarray(a).shape[0]) if not hasattr(a, "numel") else
                                int(a.shape[0]) for a in arrays])
    dist.broadcast(meta, src)
    out = []
    for k, dt in enumerate(dtypes):
        if rank == src:
            t = _upload(arrays[k], device)
        else:
            t = torch.empty(int(meta[k]), dtype=_torch_dtype(dt), device=device)
        dist.broadcast(t, src)
        out.append(t)
    return out


def scatter_arrays(blocks, dtypes, device: str):
    """Rank 0 holds `blocks[r]` (a list of arrays) for every rank r; each rank
    receives its own (point-to-point sends from rank 0; rank 0 keeps block 0)."""
    import torch

    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    n = len(dtypes)
    if rank == 0:
        for r in range(1, world):
            meta = torch.tensor([int(np.asarray(a).shape[0]) for a in blocks[r]],
                                dtype=torch.int64, device=device)
            dist.send(meta, r)
            for a in blocks[r]:
                dist.send(_upload(a, device), r)
        return [_upload(a, device) for a in blocks[0]]
    meta = torch.zeros(n, dtype=torch.int64, device=device)
    dist.recv(meta, 0)
    out = []
    for k, dt in enumerate(dtypes):
        t = torch.empty(int(meta[k]), dtype=_torch_dtype(dt), device=device)
        dist.recv(t, 0)
        out.append(t)
    return out


def broadcast_ints(vals, n: int, device: str) -> np.ndarray:
    """A small int64 vector from rank 0 (partition bounds, dimensions)."""
    import torch

    dist = _dist()
    t = torch.zeros(n, dtype=torch.int64, device=device)
    if dist.get_rank() == 0:
        t[:] = torch.as_tensor(np.asarray(vals, dtype=np.int64))
    dist.broadcast(t, 0)
    return t.cpu().numpy()


_I64, _F64 = np.int64, np.float64


def broadcast_csr(A: Optional[CSR], src: int = 0, device: str = "cpu") -> CSR:
    """A CSR from `src` to every rank (NCCL on GPUs: one transfer per array
    over NVLink/NVSwitch)."""
    dist = _dist()
    dims = broadcast_ints([A.nrows, A.ncols] if dist.get_rank() == src else None, 2, device) \
        if src == 0 else None
    pos, idx, vals = broadcast_arrays((A.pos, A.idx, A.vals) if dist.get_rank() == src else None,
                                      (_I64, _I64, _F64), src, device)
    return CSR(int(dims[0]), int(dims[1]), _out(pos, device), _out(idx, device), _out(vals, device))


def broadcast_dense(M, src: int = 0, device: str = "cpu"):
    """Dense row-major factor from `src`; returns a (rows, cols) tensor
    (numpy on "cpu")."""
    dist = _dist()
    rank = dist.get_rank()
    shape = broadcast_ints(list(np.asarray(M).shape) if rank == src and not hasattr(M, "numel")
                           else (list(M.shape) if rank == src else None), 2, device)
    (flat,) = broadcast_arrays((M.reshape(-1),) if rank == src else None, (_F64,), src, device)
    return _out(flat.view(int(shape[0]), int(shape[1])), device)


def device_rows(A: CSR, r0: int, r1: int) -> CSR:
    """Row block of a device-resident CSR as views of its idx/vals (the pos
    block is rebased: one small device subtraction, no copy of the entries)."""
    a, b = int(A.pos[r0]), int(A.pos[r1])
    pos = A.pos[r0:r1 + 1] - A.pos[r0]
    return CSR(r1 - r0, A.ncols, pos, A.idx[a:b], A.vals[a:b])


def scatter_csr_rows(A: Optional[CSR], bounds: np.ndarray, device: str) -> CSR:
    """Rank r receives rows [bounds[r], bounds[r+1]) of rank 0's A."""
    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    blocks = None
    if rank == 0:
        blocks = []
        for r in range(world):
            blk = csr_rows(A, int(bounds[r]), int(bounds[r + 1]))
            blocks.append((blk.pos, blk.idx, blk.vals))
    ncols = int(broadcast_ints([A.ncols] if rank == 0 else None, 1, device)[0])
    pos, idx, vals = scatter_arrays(blocks, (_I64, _I64, _F64), device)
    nrows = int(bounds[rank + 1] - bounds[rank])
    return CSR(nrows, ncols, _out(pos, device), _out(idx, device), _out(vals, device))


def _scatter_csf(blocks_host, dims_jk, nslices, device):
    pos1, idx1, pos2, idx2, vals = scatter_arrays(
        [(b.pos1, b.idx1, b.pos2, b.idx2, b.vals) for b in blocks_host] if blocks_host else None,
        (_I64, _I64, _I64, _I64, _F64), device)
    return CSF3((nslices, int(dims_jk[0]), int(dims_jk[1])), *(_out(t, device) for t in
                                                               (pos1, idx1, pos2, idx2, vals)))


def scatter_csf_slices(B: Optional[CSF3], bounds: np.ndarray, device: str) -> CSF3:
    """Rank r receives slices [bounds[r], bounds[r+1]) of rank 0's B."""
    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    jk = broadcast_ints(list(B.dims[1:]) if rank == 0 else None, 2, device)
    blocks = ([csf_slices(B, int(bounds[r]), int(bounds[r + 1])) for r in range(world)]
              if rank == 0 else None)
    return _scatter_csf(blocks, jk, int(bounds[rank + 1] - bounds[rank]), device)


def scatter_csf_fibers(B: Optional[CSF3], fbounds: np.ndarray, device: str):
    """Rank r receives fibers [fbounds[r], fbounds[r+1]) of rank 0's B as a CSF
    over the slices they touch.  Returns (s0, s1, sub) per rank: sub's slice 0
    is B's slice s0, and s1 - s0 = sub's slice count."""
    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    jk = broadcast_ints(list(B.dims[1:]) if rank == 0 else None, 2, device)
    if rank == 0:
        parts = [csf_fibers(B, int(fbounds[r]), int(fbounds[r + 1])) for r in range(world)]
        spans = [v for s0, sub in parts for v in (s0, s0 + sub.dims[0])]
        blocks = [sub for _, sub in parts]
    else:
        spans, blocks = None, None
    spans = broadcast_ints(spans, 2 * world, device).reshape(world, 2)
    s0, s1 = int(spans[rank, 0]), int(spans[rank, 1])
    return s0, s1, spans, _scatter_csf(blocks, jk, s1 - s0, device)


def slice_owner(spans: np.ndarray, s: int) -> int:
    """Lowest rank whose fiber block touches slice s (it owns that result row)."""
    for r in range(spans.shape[0]):
        if spans[r, 0] <= s < spans[r, 1]:
            return r
    return -1


def owned_rows(spans: np.ndarray, rank: int):
    """Local row range [a, b) of this rank's block whose slices it owns."""
    s0, s1 = int(spans[rank, 0]), int(spans[rank, 1])
    if s1 <= s0:
        return 0, 0
    a = 0 if slice_owner(spans, s0) == rank else 1
    return a, s1 - s0


def exchange_boundary_rows(part, spans: np.ndarray, device: str):
    """Adds, into the rows this rank owns, the partial first rows of the
    higher ranks whose fiber blocks start inside one of its slices (one
    all-gather of R values per rank; added in rank order, so the result does
    not depend on timing).  `part` is the rank's (rows, R) block (torch on
    "cuda", numpy on "cpu"); it is updated in place and returned."""
    import torch

    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    if world == 1:
        return part
    t = part if type(part).__module__.startswith("torch") else torch.from_numpy(part)
    R = int(t.shape[1])
    mine = torch.zeros(R, dtype=torch.float64, device=t.device)
    if t.shape[0] > 0:
        mine.copy_(t[0])
    got = [torch.empty(R, dtype=torch.float64, device=t.device) for _ in range(world)]
    dist.all_gather(got, mine)
    s_me = int(spans[rank, 0])
    for r in range(world):
        if r == rank or spans[r, 1] <= spans[r, 0]:
            continue
        s = int(spans[r, 0])
        if slice_owner(spans, s) == rank:  # r's block starts inside my slice s
            t[s - s_me] += got[r]
    return part


def distributed_spgemm(A: Optional[CSR], B: Optional[CSR], compute: Callable[[CSR, CSR], CSR],
                       device: str = "cpu", gather: bool = False, same: bool = False):
    """Row-sharded C = A·B.  Rank 0 holds A and B; B is broadcast once, each
    rank computes its product-balanced row block of A (a view of the broadcast
    copy when `same`, i.e. B is A).  Returns (row0, C_shard) and, with
    gather=True, the global CSR on every rank."""
    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    bounds = broadcast_ints(balanced_bounds(spgemm_row_weights(A, B), world) if rank == 0 else None,
                            world + 1, device)
    Bb = broadcast_csr(B if rank == 0 else None, 0, device)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    Al = (device_rows(Bb, r0, r1) if device != "cpu" else csr_rows(Bb, r0, r1)) if same \
        else scatter_csr_rows(A, bounds, device)
    part = compute(Al, Bb)
    if not gather:
        return r0, part
    parts = [None] * world
    dist.all_gather_object(parts, part.numpy())
    return r0, concat_csr(parts)


def distributed_spadd(ops: Optional[Sequence[CSR]], compute: Callable[[Sequence[CSR]], CSR],
                      device: str = "cpu", gather: bool = False):
    """Row-sharded D = sum(ops): row i of D depends only on row i of every
    operand, so each rank adds its nnz-balanced row block; no collective on
    the data path (rank 0 scatters the blocks once).  Returns (row0, D_shard)
    and, with gather=True, the global CSR on every rank."""
    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    nops = int(broadcast_ints([len(ops)] if rank == 0 else None, 1, device)[0])
    w = sum(np.diff(_np(o.pos)) for o in ops) if rank == 0 else None
    bounds = broadcast_ints(balanced_bounds(w, world) if rank == 0 else None, world + 1, device)
    local = [scatter_csr_rows(ops[q] if rank == 0 else None, bounds, device) for q in range(nops)]
    r0 = int(bounds[rank])
    part = compute(local)
    if not gather:
        return r0, part
    parts = [None] * world
    dist.all_gather_object(parts, part.numpy())
    return r0, concat_csr(parts)


def distributed_mttkrp_dense(B: Optional[CSF3], C, D, compute: Callable, device: str = "cpu"):
    """A = B x_2 C x_3 D with a dense result over fiber-balanced blocks.  The
    factors are broadcast once; each rank computes the rows of the slices its
    fibers touch, then one all-gather of the first partial rows completes the
    cut slices (exchange_boundary_rows).  Returns the full A on every rank
    (assembled from the owned row ranges; test/inspection path)."""
    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    fb = broadcast_ints(fiber_bounds(B, world) if rank == 0 else None, world + 1, device)
    Cf = broadcast_dense(C if rank == 0 else None, 0, device)
    Df = broadcast_dense(D if rank == 0 else None, 0, device)
    I = int(broadcast_ints([B.dims[0]] if rank == 0 else None, 1, device)[0])
    s0, s1, spans, sub = scatter_csf_fibers(B, fb, device)
    R = int(Cf.shape[1])
    if sub.dims[0] > 0:
        part = compute(sub, Cf, Df)
        part = np.asarray(part, dtype=np.float64).reshape(sub.dims[0], R) if device == "cpu" \
            else part
    else:
        part = np.zeros((0, R)) if device == "cpu" else None
    part = exchange_boundary_rows(part if part is not None else _empty_rows(R, device), spans,
                                  device)
    a, b = owned_rows(spans, rank)
    blocks = [None] * world
    dist.all_gather_object(blocks, (s0 + a, np.asarray(_np(part[a:b])).reshape(b - a, R)))
    A = np.zeros((I, R))
    for s, blk in blocks:
        if blk.size:
            A[s:s + blk.shape[0]] = blk
    return A


def _empty_rows(R, device):
    import torch

    return torch.zeros((0, R), dtype=torch.float64, device=device)


def distributed_mttkrp_sparse(B: Optional[CSF3], C: Optional[CSR], D: Optional[CSR],
                              compute: Callable[[CSF3, CSR, CSR], CSR], device: str = "cpu",
                              gather: bool = False):
    """Sparse-result MTTKRP over nnz-balanced i-slice blocks (slice-aligned:
    a result row is a compacted workspace, so a slice is not split); factors
    broadcast once, results stay row-sharded.  Returns (slice0, A_shard) and,
    with gather=True, the global CSR."""
    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size()
    if rank == 0:
        pos1, pos2 = _np(B.pos1), _np(B.pos2)
        bounds = balanced_bounds(np.diff(pos2[pos1]), world)  # nnz per slice
    bounds = broadcast_ints(bounds if rank == 0 else None, world + 1, device)
    Cf = broadcast_csr(C if rank == 0 else None, 0, device)
    Df = broadcast_csr(D if rank == 0 else None, 0, device)
    sub = scatter_csf_slices(B, bounds, device)
    i0 = int(bounds[rank])
    part = compute(sub, Cf, Df)
    if not gather:
        return i0, part
    parts = [None] * world
    dist.all_gather_object(parts, part.numpy())
    return i0, concat_csr(parts)
