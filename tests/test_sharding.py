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
        r0, C = S.distributed_spgemm(A, A, lambda a, b: compute(a.numpy(), b.numpy()),
                                     gather=True, same=True)
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


def _worker_more(rank, world, port, q):
    """SpAdd, dense MTTKRP (fiber-balanced, heavy slice cut between ranks) and
    sparse MTTKRP (slice-aligned) through the N>1 orchestration on gloo."""
    import torch.distributed as dist

    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        def as_csr(o):
            return CSR(o["nrows"], o["ncols"], o["pos"], o["idx"], o["vals"])

        c2 = G.make_config(2, scale=0.002) if rank == 0 else None
        _, D = S.distributed_spadd(c2["ops"] if c2 else None, lambda ops: as_csr(oracle.spadd([o.numpy() for o in ops])),
                                   gather=True)
        c4 = G.make_config(4, scale=0.003) if rank == 0 else None
        A4 = S.distributed_mttkrp_dense(
            c4["B"] if c4 else None, c4["C"].vals if c4 else None, c4["D"].vals if c4 else None,
            lambda b, c, d: oracle.mttkrp_dense(b, c, d)["vals"] if b.dims[0] else
            np.zeros((0, c.shape[1])))
        c5 = G.make_config(5, scale=0.0005) if rank == 0 else None
        _, A5 = S.distributed_mttkrp_sparse(c5["B"] if c5 else None, c5["C"] if c5 else None,
                                            c5["D"] if c5 else None,
                                            lambda b, c, d: as_csr(oracle.mttkrp_sparse(b, c, d)),
                                            gather=True)
        if rank == 0:
            r2 = oracle.spadd(c2["ops"])
            out["spadd"] = bool(np.array_equal(D.pos, r2["pos"]) and np.array_equal(D.idx, r2["idx"])
                                and np.array_equal(D.vals.view(np.int64), r2["vals"].view(np.int64)))
            r4 = oracle.mttkrp_dense(c4["B"], c4["C"].vals, c4["D"].vals)
            bound = 1e-12 * np.maximum(np.abs(r4["vals"]), r4["abs"])
            out["mttkrp_dense"] = bool(np.all(np.abs(A4 - r4["vals"]) <= bound))
            # the fiber split really cuts a slice between the ranks
            fb = S.fiber_bounds(c4["B"], world)
            pos1 = np.asarray(c4["B"].pos1)
            out["cut_inside_slice"] = bool(not np.isin(fb[1:-1], pos1).all())
            r5 = oracle.mttkrp_sparse(c5["B"], c5["C"], c5["D"])
            out["mttkrp_sparse"] = bool(np.array_equal(A5.pos, r5["pos"]) and
                                        np.array_equal(A5.idx, r5["idx"]) and
                                        np.array_equal(A5.vals.view(np.int64),
                                                       r5["vals"].view(np.int64)))
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_distributed_spadd_and_mttkrp_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_more, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = q.get(timeout=5)
    assert res == {"spadd": True, "mttkrp_dense": True, "cut_inside_slice": True,
                   "mttkrp_sparse": True}, res


def test_csf_fibers_partial_slices_sum_to_the_whole():
    import oracle

    cfg = G.make_config(4, scale=0.003)
    B, Cv, Dv = cfg["B"], cfg["C"].vals, cfg["D"].vals
    ref = oracle.mttkrp_dense(B, Cv, Dv)
    for parts in (2, 3, 7):
        fb = S.fiber_bounds(B, parts)
        A = np.zeros_like(ref["vals"])
        for p in range(parts):
            s0, sub = S.csf_fibers(B, int(fb[p]), int(fb[p + 1]))
            sub.validate()
            if sub.dims[0]:
                A[s0:s0 + sub.dims[0]] += oracle.mttkrp_dense(sub, Cv, Dv)["vals"]
        assert np.all(np.abs(A - ref["vals"]) <= 1e-12 * np.maximum(np.abs(ref["vals"]), ref["abs"]))


def _worker_dense3(rank, world, port, q):
    """Dense MTTKRP over 3 ranks whose fiber blocks cut the heaviest slice:
    the boundary-row all-gather completes every cut slice (one slice spans
    all three blocks here)."""
    import torch.distributed as dist

    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B = None
        if rank == 0:
            sizes = np.array([3000, 10, 10, 5, 5, 3, 2, 1], dtype=np.int64)  # one dominant slice
            B = G.csf3((8, 60, 80), sizes, 91)
            Cm, Dm = G.dense(60, 8, 92).vals, G.dense(80, 8, 93).vals
        A = S.distributed_mttkrp_dense(B, Cm if rank == 0 else None, Dm if rank == 0 else None,
                                       lambda b, c, d: oracle.mttkrp_dense(b, c, d)["vals"])
        if rank == 0:
            fb = S.fiber_bounds(B, world)
            spans = [S.csf_fibers(B, int(fb[r]), int(fb[r + 1]))[0] for r in range(world)]
            r = oracle.mttkrp_dense(B, Cm, Dm)
            ok = bool(np.all(np.abs(A - r["vals"]) <= 1e-12 * np.maximum(np.abs(r["vals"]), r["abs"])))
            q.put({"ok": ok, "all_start_in_slice0": spans == [0, 0, 0]})
    finally:
        dist.destroy_process_group()


def test_distributed_mttkrp_dense_slice_spanning_three_ranks_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_dense3, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = q.get(timeout=5)
    assert res == {"ok": True, "all_start_in_slice0": True}, res
