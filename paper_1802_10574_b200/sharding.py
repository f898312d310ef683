"""Multi-GPU sharding of the hot path: one process per GPU,
``torch.distributed`` (NCCL over NVLink/NVSwitch on GPUs, gloo on CPU for tests).

Every kernel shards without a data-path reduction:

* SpGEMM  — contiguous row blocks of A balanced by the prefix of per-row
  products (sum over A(i,:) of nnz(B_k)); B is broadcast once from rank 0.
* SpAdd   — contiguous row blocks balanced by operand nnz; nothing broadcast.
* MTTKRP  — contiguous i-slice blocks balanced by nnz; factors broadcast once.

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
