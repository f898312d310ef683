"""Multi-GPU sharding of the hot path: one process per GPU,
``torch.distributed`` (NCCL over NVLink/NVSwitch on GPUs, gloo on CPU for tests).

Every kernel shards without a data-path reduction:

* SpGEMM  — contiguous row blocks of A balanced by the prefix of per-row
  products (sum over A(i,:) of nnz(B_k)); B is broadcast once from rank 0.
* SpAdd   — contiguous row blocks balanced by operand nnz; nothing broadcast.
* MTTKRP  — factors broadcast once.  Dense result: contiguous fiber blocks
  balanced by nnz (cut inside slices: config 4's heaviest slice holds 38.5 %
  of the nonzeros); the only exchange is the partial rows of the <= N-1 cut
  slices, summed in rank order.  Sparse result: nnz-balanced i-slice blocks
  (slice-aligned; a result row is one compacted workspace).

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


# ---------------------------------------------------------------------------
# collectives (torch.distributed): broadcast once, gather shard sizes
# ---------------------------------------------------------------------------
def broadcast_csr(A: Optional[CSR], src: int = 0, device: str = "cpu") -> CSR:
    """Broadcast a CSR from `src` to every rank (NCCL on GPUs: one transfer per
    array over NVLink/NVSwitch)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank()
    meta = torch.zeros(3, dtype=torch.int64, device=device)
    if rank == src:
        meta[:] = torch.tensor([A.nrows, A.ncols, A.nnz])
    dist.broadcast(meta, src)
    nrows, ncols, nnz = (int(x) for x in meta.tolist())
    out = []
    for k, (n, dt) in enumerate(((nrows + 1, torch.int64), (nnz, torch.int64),
                                 (nnz, torch.float64))):
        if rank == src:
            t = torch.as_tensor(_np((A.pos, A.idx, A.vals)[k])).to(device)
        else:
            t = torch.empty(n, dtype=dt, device=device)
        dist.broadcast(t, src)
        out.append(t if device != "cpu" else t.numpy())
    return CSR(nrows, ncols, *out)


def distributed_spgemm(A: Optional[CSR], B: Optional[CSR], compute: Callable[[CSR, CSR], CSR],
                       device: str = "cpu", gather: bool = False):
    """Row-sharded C = A·B.  Rank 0 holds A and B; B is broadcast once, each
    rank computes its product-balanced row block.  Returns (row0, C_shard) and,
    with gather=True, the global CSR on rank 0."""
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    Bb = broadcast_csr(B if rank == 0 else None, 0, device)
    Ab = broadcast_csr(A if rank == 0 else None, 0, device)
    Bh = CSR(Bb.nrows, Bb.ncols, _np(Bb.pos), _np(Bb.idx), _np(Bb.vals))
    Ah = CSR(Ab.nrows, Ab.ncols, _np(Ab.pos), _np(Ab.idx), _np(Ab.vals))
    bounds = balanced_bounds(spgemm_row_weights(Ah, Bh), world)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    part = compute(csr_rows(Ah, r0, r1), Bb if device != "cpu" else Bh)
    if not gather:
        return r0, part
    parts = [None] * world
    dist.all_gather_object(parts, CSR(part.nrows, part.ncols, _np(part.pos), _np(part.idx),
                                      _np(part.vals)))
    return r0, concat_csr(parts)


# ---------------------------------------------------------------------------
# SpAdd and MTTKRP
# ---------------------------------------------------------------------------
def broadcast_csf(B: Optional[CSF3], src: int = 0, device: str = "cpu") -> CSF3:
    """Broadcast a CSF(3) from `src` (one transfer per level array)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank()
    meta = torch.zeros(5, dtype=torch.int64, device=device)
    if rank == src:
        meta[:] = torch.tensor([*B.dims, B.nfibers, B.nnz])
    dist.broadcast(meta, src)
    I, J, K, nf, nnz = (int(x) for x in meta.tolist())
    shapes = ((I + 1, torch.int64), (nf, torch.int64), (nf + 1, torch.int64),
              (nnz, torch.int64), (nnz, torch.float64))
    out = []
    for k, (n, dt) in enumerate(shapes):
        if rank == src:
            t = torch.as_tensor(_np((B.pos1, B.idx1, B.pos2, B.idx2, B.vals)[k])).to(device)
        else:
            t = torch.empty(n, dtype=dt, device=device)
        dist.broadcast(t, src)
        out.append(t if device != "cpu" else t.numpy())
    return CSF3((I, J, K), *out)


def broadcast_dense(M: Optional[np.ndarray], src: int = 0, device: str = "cpu"):
    import torch
    import torch.distributed as dist

    rank = dist.get_rank()
    meta = torch.zeros(2, dtype=torch.int64, device=device)
    if rank == src:
        meta[:] = torch.tensor(list(np.asarray(M).shape))
    dist.broadcast(meta, src)
    r, c = (int(x) for x in meta.tolist())
    t = (torch.as_tensor(np.ascontiguousarray(M)).to(device) if rank == src
         else torch.empty((r, c), dtype=torch.float64, device=device))
    dist.broadcast(t, src)
    return t if device != "cpu" else t.numpy()


def distributed_spadd(ops: Optional[Sequence[CSR]], compute: Callable[[Sequence[CSR]], CSR],
                      device: str = "cpu", gather: bool = False):
    """Row-sharded D = sum(ops): row i of D depends only on row i of every
    operand, so each rank adds its nnz-balanced row block; no data-path
    collective (the operands are broadcast here only because rank 0 holds
    them in the test harness).  Returns (row0, D_shard) and, with gather=True,
    the global CSR on every rank."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    n = torch.zeros(1, dtype=torch.int64)
    if rank == 0:
        n[0] = len(ops)
    dist.broadcast(n, 0)
    full = [broadcast_csr(ops[q] if rank == 0 else None, 0, "cpu") for q in range(int(n[0]))]
    w = sum(np.diff(_np(o.pos)) for o in full)
    bounds = balanced_bounds(w, world)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    part = compute([csr_rows(o, r0, r1) for o in full])
    if not gather:
        return r0, part
    parts = [None] * world
    dist.all_gather_object(parts, CSR(part.nrows, part.ncols, _np(part.pos), _np(part.idx),
                                      _np(part.vals)))
    return r0, concat_csr(parts)


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


def distributed_mttkrp_dense(B: Optional[CSF3], C: Optional[np.ndarray], D: Optional[np.ndarray],
                             compute: Callable[[CSF3, np.ndarray, np.ndarray], np.ndarray],
                             device: str = "cpu"):
    """A = B x_2 C x_3 D with a dense result over fiber-balanced blocks.  The
    factors are broadcast once; each rank computes the rows of the slices its
    fibers touch.  A slice cut between ranks leaves partial rows on both: the
    only exchange is those boundary rows (at most world - 1 slices), summed on
    every rank in rank order (deterministic).  Returns the full A on every
    rank."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    Bf = broadcast_csf(B if rank == 0 else None, 0, "cpu")
    Cf = broadcast_dense(C if rank == 0 else None, 0, device)
    Df = broadcast_dense(D if rank == 0 else None, 0, device)
    fb = fiber_bounds(Bf, world)
    s0, sub = csf_fibers(Bf, int(fb[rank]), int(fb[rank + 1]))
    part = np.asarray(_np(compute(sub, Cf, Df)), dtype=np.float64).reshape(sub.dims[0], -1)
    R = part.shape[1] if part.size else _np(Cf).shape[1]
    # every rank's block and its first slice; rows are disjoint except at cuts
    blocks = [None] * world
    dist.all_gather_object(blocks, (s0, part))
    A = np.zeros((Bf.dims[0], R))
    for s, blk in blocks:  # rank order: boundary rows add in a fixed order
        if blk.size:
            A[s:s + blk.shape[0]] += blk
    return A


def distributed_mttkrp_sparse(B: Optional[CSF3], C: Optional[CSR], D: Optional[CSR],
                              compute: Callable[[CSF3, CSR, CSR], CSR], device: str = "cpu",
                              gather: bool = False):
    """Sparse-result MTTKRP over nnz-balanced i-slice blocks (slice-aligned:
    a result row is a compacted workspace, so a slice is not split); factors
    broadcast once, results stay row-sharded.  Returns (slice0, A_shard) and,
    with gather=True, the global CSR."""
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    Bf = broadcast_csf(B if rank == 0 else None, 0, "cpu")
    Cf = broadcast_csr(C if rank == 0 else None, 0, device)
    Df = broadcast_csr(D if rank == 0 else None, 0, device)
    pos1, pos2 = _np(Bf.pos1), _np(Bf.pos2)
    w = np.diff(pos2[pos1])  # nnz per slice
    bounds = balanced_bounds(w, world)
    i0, i1 = int(bounds[rank]), int(bounds[rank + 1])
    part = compute(csf_slices(Bf, i0, i1), Cf, Df)
    if not gather:
        return i0, part
    parts = [None] * world
    dist.all_gather_object(parts, CSR(part.nrows, part.ncols, _np(part.pos), _np(part.idx),
                                      _np(part.vals)))
    return i0, concat_csr(parts)
