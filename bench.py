#!/usr/bin/env python
"""Benchmark of the hot path.

One "step" = one call of the kernel entry point (C ABI) over one batch of
synthetic input with BASELINE.json's shapes.  With no ``--config`` every one of
BASELINE's five configs is measured and reported in ``configs``; the headline
fields (``value``, ``roofline``, ``e2e``, ``cpu_baseline``) are those of the
largest single-GPU config, config 5 (sparse-result MTTKRP, 7.2 GB per call).
``--config K`` measures config K alone and makes it the headline.

Our arm (default):
  value    = algorithmic HBM bytes of the call (inputs read once + output written
             once, int64 indices / fp64 values) / device time per step, with the
             inputs resident in HBM; whole-job aggregate over ranks.
  e2e      = the same metric through the same C-ABI call with pinned HOST
             inputs and a HOST result (H2D + D2H inside the timed region).
  roofline = the call's algorithmic bytes / its kernels' CUDA-event durations
             vs the measured HBM copy bandwidth (MEASURED_PEAKS.json).
  cpu_baseline = the reference CPU path (oracle/_ref: the reference's own
             Workspace/TensorBuilder) on the host: 1 thread (SPEC.md:425-426,
             PAPER.md:1484-1486) and all host threads, median of 5 after a
             discarded warm-up, bounded row/slice sample.

``--impl reference``: rank 0 times the reference CPU path alone on the
headline config/metric (other ranks exit), printing the same JSON line.

Multi-GPU (torchrun, N ranks): STRONG scaling on one problem.  Rank 0
generates the problem; the operand every rank reads in full (SpGEMM's B, the
MTTKRP factors) is broadcast once over NCCL (``broadcast_ms``, outside the
step), row / fiber / slice blocks are scattered once (sharding.py); a step is
every rank's call on its block (+ the dense MTTKRP's boundary-row all-gather);
time = max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

L2_BYTES = 126e6
METRIC = "SpGEMM/SpAdd/MTTKRP useful GFLOP/s; achieved HBM GB/s vs B200 peak"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback if MEASURED_PEAKS.json is absent
HEADLINE = 5               # largest single-GPU config (7.2 GB algorithmic per call)


def _peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def _traffic(workload: str, kernel: str):
    """DRAM bytes per launch from a committed `ncu --set full` capture."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        d = json.loads(p.read_text())
        return d.get(workload, {}).get(kernel)
    except Exception:
        return None


def _csr_bytes(m) -> int:
    return 8 * (m.nrows + 1) + 16 * m.nnz


def _csf_bytes(b) -> int:
    return 8 * (b.dims[0] + 1) + 8 * b.nfibers + 8 * (b.nfibers + 1) + 16 * b.nnz


def _pin(a):
    """Pinned host copy of a (host or device) array."""
    import torch

    t = a if type(a).__module__.startswith("torch") else torch.from_numpy(np.ascontiguousarray(a))
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h


def _sync():
    import torch

    torch.cuda.synchronize()


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
class Workload:
    """Inputs on device (the rank's block), raw C-ABI step, e2e step, CPU ref.

    Rank 0 generates the whole problem (``cfg``); ``distribute`` leaves every
    rank with its block resident on its GPU (``dist_on`` False: one process,
    the whole problem)."""

    mode = "fused"  # fused | assemble | compute | unsorted (SpGEMM, SpAdd)

    def __init__(self, cid: int, have_data: bool = True):
        from paper_1802_10574_b200 import generators as G

        self.cid = cid
        self.name = G.CONFIG_NAMES[cid]
        self.cfg = None
        self.gen_s = 0.0
        if have_data:
            t = time.time()
            self.cfg = G.make_config(cid)
            self.gen_s = time.time() - t
        self.broadcast_ms = 0.0
        self.broadcast_bytes = 0

    def _bcast(self, fn):
        """Runs a broadcast, timing it (device-synchronised wall clock)."""
        _sync()
        t = time.perf_counter()
        out = fn()
        _sync()
        self.broadcast_ms += (time.perf_counter() - t) * 1e3
        return out

    def _init_native(self, ctx):
        from paper_1802_10574_b200 import _native as N

        self.N, self.ctx, self.lib = N, ctx, N.load()

    def release(self, r):
        self.N.check(self.lib.stam_cuda_release(self.ctx._ctx, C.c_void_p(r.handle)))

    def post_step(self, r):
        """Data-path exchange after the call (dense MTTKRP at N > 1)."""

    def algo_bytes_total(self, dist_on):
        """Whole-problem algorithmic bytes: every rank's own block inputs and
        outputs + the broadcast operand once."""
        own = self.own_in_bytes + self.out_bytes
        if dist_on:
            import torch
            import torch.distributed as dist

            t = torch.tensor([float(own)], dtype=torch.float64, device="cuda")
            dist.all_reduce(t)
            own = float(t.item())
        return own + self.shared_bytes


class SpaddWork(Workload):
    def distribute(self, world, rank, dist_on):
        from paper_1802_10574_b200 import sharding as S

        if not dist_on:
            self.local = [o.to("cuda") for o in self.cfg["ops"]]
        else:
            ops = self.cfg["ops"] if rank == 0 else None
            nops = int(S.broadcast_ints([len(ops)] if rank == 0 else None, 1, "cuda")[0])
            w = sum(np.diff(o.pos) for o in ops) if rank == 0 else None
            bounds = S.broadcast_ints(S.balanced_bounds(w, world) if rank == 0 else None,
                                      world + 1, "cuda")
            self.local = [S.scatter_csr_rows(ops[q] if rank == 0 else None, bounds, "cuda")
                          for q in range(nops)]
            self.row0 = int(bounds[rank])
        self.own_in_bytes = sum(_csr_bytes(o) for o in self.local)
        self.shared_bytes = 0
        self.local_adds = sum(o.nnz for o in self.local[1:])

    def setup(self, ctx):
        from paper_1802_10574_b200.storage import CSR

        self._init_native(ctx)
        N = self.N
        self.views = (N.CsrView * len(self.local))(*[o.view() for o in self.local])
        self.hops = [CSR(o.nrows, o.ncols, _pin(o.pos), _pin(o.idx), _pin(o.vals))
                     for o in self.local]
        self.hviews = (N.CsrView * len(self.hops))(*[h.view() for h in self.hops])
        self.nnz_out = None

    def _index(self, views):
        """Pre-assembled index for compute mode (assembled once, reused)."""
        if getattr(self, "_idx", None) is None:
            N = self.N
            r = N.CsrResult()
            opts = N.Options(1, N.STAM_MODE_ASSEMBLE, N.STAM_MEM_DEVICE, 0)
            N.check(self.lib.stam_cuda_spadd(self.ctx._ctx, len(self.local), self.views,
                                             C.byref(opts), C.byref(r), C.byref(N.Stats())))
            self._idx = r
            self._idx_view = N.CsrView(r.nrows, r.ncols, r.nnz, r.pos, r.idx, r.vals,
                                       N.STAM_MEM_DEVICE, 0)
        return self._idx_view

    def _call(self, views, result_mem, timing):
        N = self.N
        r = N.CsrResult()
        st = N.Stats()
        mode = {"assemble": N.STAM_MODE_ASSEMBLE, "compute": N.STAM_MODE_COMPUTE}.get(
            self.mode, N.STAM_MODE_FUSED)
        opts = N.Options(0 if self.mode == "unsorted" else 1, mode, result_mem,
                         1 if timing else 0)
        if self.mode == "compute":
            N.check(self.lib.stam_cuda_spadd_compute(
                self.ctx._ctx, len(self.local), views, C.byref(self._index(views)),
                C.byref(opts), C.byref(r), C.byref(st)))
        else:
            N.check(self.lib.stam_cuda_spadd(self.ctx._ctx, len(self.local), views,
                                             C.byref(opts), C.byref(r), C.byref(st)))
        self.nnz_out = r.nnz
        self.out_bytes = 8 * (r.nrows + 1) + 16 * r.nnz
        self.release(r)
        return st

    def step(self, timing=False):
        return self._call(self.views, self.N.STAM_MEM_DEVICE, timing)

    def e2e_step(self):
        return self._call(self.hviews, self.N.STAM_MEM_HOST, False)

    def local_flops(self):
        # workspace adds executed (SPEC counters: every accumulate insert)
        return self.local_adds

    def h2d_bytes(self):
        return self.own_in_bytes

    def d2h_bytes(self):
        return self.out_bytes

    # reference CPU path on a row sample (rank 0, whole problem)
    def total_units(self):
        return self.cfg["ops"][0].nrows

    def ref_sample(self, rows):
        from paper_1802_10574_b200.storage import CSR

        sub = []
        for o in self.cfg["ops"]:
            e = int(o.pos[rows])
            sub.append(CSR(rows, o.ncols, o.pos[: rows + 1], o.idx[:e], o.vals[:e]))
        return sub

    def ref_run(self, sample, nthreads):
        import oracle

        out = oracle.ref_spadd(sample, nthreads)
        return sum(_csr_bytes(o) for o in sample) + 8 * (out["nrows"] + 1) + 16 * int(
            out["pos"][-1]), sum(o.nnz for o in sample[1:])


class SpgemmWork(Workload):
    """C = A*B (configs 1 and 3; config 3 squares A, so B is A)."""

    def distribute(self, world, rank, dist_on):
        import torch

        from paper_1802_10574_b200 import sharding as S

        if not dist_on:
            A, B = self.cfg["A"], self.cfg["B"]
            self.same = B is A
            self.Al = A.to("cuda")
            self.Bd = self.Al if self.same else B.to("cuda")
            self.own_in_bytes = _csr_bytes(A)
            self.shared_bytes = 0 if self.same else _csr_bytes(B)
        else:
            A = self.cfg["A"] if rank == 0 else None
            B = self.cfg["B"] if rank == 0 else None
            self.same = bool(S.broadcast_ints([int(B is A)] if rank == 0 else None, 1, "cuda")[0])
            bounds = S.broadcast_ints(
                S.balanced_bounds(S.spgemm_row_weights(A, B), world) if rank == 0 else None,
                world + 1, "cuda")
            # B broadcast once over NVLink (for A·A this is A itself)
            self.Bd = self._bcast(lambda: S.broadcast_csr(B, 0, "cuda"))
            self.broadcast_bytes = _csr_bytes(self.Bd)
            r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
            self.row0 = r0
            self.Al = (S.device_rows(self.Bd, r0, r1) if self.same
                       else S.scatter_csr_rows(A, bounds, "cuda"))
            # A·A: A's bytes are the broadcast operand's (counted once)
            self.own_in_bytes = 0 if self.same else _csr_bytes(self.Al)
            self.shared_bytes = _csr_bytes(self.Bd)
        blen = self.Bd.pos[1:] - self.Bd.pos[:-1]
        self.local_products = int(blen[self.Al.idx].sum().item()) if self.Al.nnz else 0
        torch.cuda.synchronize()

    def setup(self, ctx):
        from paper_1802_10574_b200.storage import CSR

        self._init_native(ctx)
        self.va, self.vb = self.Al.view(), self.Bd.view()
        pin = lambda m: CSR(m.nrows, m.ncols, _pin(m.pos), _pin(m.idx), _pin(m.vals))
        self.Ah = pin(self.Al)
        self.Bh = self.Ah if (self.same and self.Al.nrows == self.Bd.nrows) else pin(self.Bd)
        self.ha, self.hb = self.Ah.view(), self.Bh.view()
        self.nnz_out = None

    def _index(self):
        """Pre-assembled index for compute mode (assembled once, reused)."""
        if getattr(self, "_idx", None) is None:
            N = self.N
            r = N.CsrResult()
            opts = N.Options(1, N.STAM_MODE_ASSEMBLE, N.STAM_MEM_DEVICE, 0)
            N.check(self.lib.stam_cuda_spgemm(self.ctx._ctx, C.byref(self.va), C.byref(self.vb),
                                              C.byref(opts), C.byref(r), C.byref(N.Stats())))
            self._idx = r
            self._idx_view = N.CsrView(r.nrows, r.ncols, r.nnz, r.pos, r.idx, r.vals,
                                       N.STAM_MEM_DEVICE, 0)
        return self._idx_view

    def _call(self, va, vb, result_mem, timing):
        N = self.N
        r = N.CsrResult()
        st = N.Stats()
        mode = {"assemble": N.STAM_MODE_ASSEMBLE, "compute": N.STAM_MODE_COMPUTE}.get(
            self.mode, N.STAM_MODE_FUSED)
        opts = N.Options(0 if self.mode == "unsorted" else 1, mode, result_mem,
                         1 if timing else 0)
        if self.mode == "compute":
            N.check(self.lib.stam_cuda_spgemm_compute(self.ctx._ctx, C.byref(va), C.byref(vb),
                                                      C.byref(self._index()), C.byref(opts),
                                                      C.byref(r), C.byref(st)))
        else:
            N.check(self.lib.stam_cuda_spgemm(self.ctx._ctx, C.byref(va), C.byref(vb),
                                              C.byref(opts), C.byref(r), C.byref(st)))
        self.nnz_out = r.nnz
        self.out_bytes = 8 * (r.nrows + 1) + 16 * r.nnz
        self.release(r)
        return st

    def step(self, timing=False):
        return self._call(self.va, self.vb, self.N.STAM_MEM_DEVICE, timing)

    def e2e_step(self):
        return self._call(self.ha, self.hb, self.N.STAM_MEM_HOST, False)

    def local_flops(self):
        return 2 * self.local_products

    def h2d_bytes(self):
        return _csr_bytes(self.Al) + (0 if self.Bh is self.Ah else _csr_bytes(self.Bd))

    def d2h_bytes(self):
        return self.out_bytes

    def total_units(self):
        return self.cfg["A"].nrows

    def ref_sample(self, rows):
        from paper_1802_10574_b200.storage import CSR

        A = self.cfg["A"]
        e = int(A.pos[rows])
        return (CSR(rows, A.ncols, A.pos[: rows + 1], A.idx[:e], A.vals[:e]), self.cfg["B"])

    def ref_run(self, sample, nthreads):
        import oracle

        A, B = sample
        out = oracle.ref_spgemm(A, B, nthreads)
        same = self.cfg["B"] is self.cfg["A"]
        nbytes = _csr_bytes(A) + (0 if same else _csr_bytes(B)) + 8 * (out["nrows"] + 1) + \
            16 * int(out["pos"][-1])
        return nbytes, 2 * int(np.sum(np.diff(B.pos)[A.idx]))


class MttkrpWork(Workload):
    """A = B x_2 C x_3 D: dense factors (config 4) or CSR factors (config 5)."""

    def distribute(self, world, rank, dist_on):
        import torch

        from paper_1802_10574_b200 import sharding as S
        from paper_1802_10574_b200.storage import Dense

        self.dist_on = dist_on
        if not dist_on:
            B, Cf, Df = self.cfg["B"], self.cfg["C"], self.cfg["D"]
            self.dense = isinstance(Cf, Dense)
            self.Bl, self.Cd, self.Dd = B.to("cuda"), Cf.to("cuda"), Df.to("cuda")
            self.spans = None
        else:
            cfg = self.cfg
            self.dense = bool(S.broadcast_ints(
                [int(isinstance(cfg["C"], Dense))] if rank == 0 else None, 1, "cuda")[0])
            B = cfg["B"] if rank == 0 else None
            if self.dense:
                fb = S.broadcast_ints(S.fiber_bounds(B, world) if rank == 0 else None,
                                      world + 1, "cuda")
                self.Cd = Dense(self._bcast(lambda: S.broadcast_dense(
                    cfg["C"].vals if rank == 0 else None, 0, "cuda")))
                self.Dd = Dense(self._bcast(lambda: S.broadcast_dense(
                    cfg["D"].vals if rank == 0 else None, 0, "cuda")))
                self.s0, _, self.spans, self.Bl = S.scatter_csf_fibers(B, fb, "cuda")
            else:
                if rank == 0:
                    pos1, pos2 = B.pos1, B.pos2
                    bounds = S.balanced_bounds(np.diff(pos2[pos1]), world)
                bounds = S.broadcast_ints(bounds if rank == 0 else None, world + 1, "cuda")
                self.Cd = self._bcast(lambda: S.broadcast_csr(cfg["C"] if rank == 0 else None,
                                                               0, "cuda"))
                self.Dd = self._bcast(lambda: S.broadcast_csr(cfg["D"] if rank == 0 else None,
                                                               0, "cuda"))
                self.Bl = S.scatter_csf_slices(B, bounds, "cuda")
                self.spans = None
                self.s0 = int(bounds[rank])
        if self.dense:
            self.R = int(self.Cd.vals.shape[1])
            self.shared_bytes = 8 * (self.Cd.vals.numel() + self.Dd.vals.numel())
            self.useful = 2 * self.R * (self.Bl.nnz + self.Bl.nfibers)
            # every nonzero reads a factor row of D and every fiber one of C:
            # the loop nest's operand stream from L2
            self.l2_gather = 8 * self.R * (self.Bl.nnz + self.Bl.nfibers)
        else:
            self.R = self.Cd.ncols
            self.shared_bytes = _csr_bytes(self.Cd) + _csr_bytes(self.Dd)
            self.useful = None
        self.broadcast_bytes = self.shared_bytes if dist_on else 0
        self.own_in_bytes = _csf_bytes(self.Bl)
        torch.cuda.synchronize()

    def setup(self, ctx):
        from paper_1802_10574_b200.storage import CSF3, CSR, Dense

        self._init_native(ctx)
        self.vB, self.vC, self.vD = self.Bl.view(), self.Cd.view(), self.Dd.view()
        B = self.Bl
        self.Bh = CSF3(B.dims, *[_pin(a) for a in (B.pos1, B.idx1, B.pos2, B.idx2, B.vals)])
        if self.dense:
            self.Ch, self.Dh = Dense(_pin(self.Cd.vals)), Dense(_pin(self.Dd.vals))
        else:
            self.Ch = CSR(self.Cd.nrows, self.Cd.ncols,
                          *[_pin(a) for a in (self.Cd.pos, self.Cd.idx, self.Cd.vals)])
            self.Dh = CSR(self.Dd.nrows, self.Dd.ncols,
                          *[_pin(a) for a in (self.Dd.pos, self.Dd.idx, self.Dd.vals)])
        self.hB, self.hC, self.hD = self.Bh.view(), self.Ch.view(), self.Dh.view()
        self.nnz_out = None

    def _call(self, vB, vC, vD, result_mem, timing):
        N = self.N
        st = N.Stats()
        opts = N.Options(1, 0, result_mem, 1 if timing else 0)
        if self.dense:
            r = N.DenseResult()
            N.check(self.lib.stam_cuda_mttkrp_dense(self.ctx._ctx, C.byref(vB), C.byref(vC),
                                                    C.byref(vD), C.byref(opts), C.byref(r),
                                                    C.byref(st)))
            self.out_bytes = 8 * r.nrows * r.ncols
            self.nnz_out = r.nrows * r.ncols
            if result_mem == N.STAM_MEM_DEVICE:
                self.post_step(r)
        else:
            r = N.CsrResult()
            N.check(self.lib.stam_cuda_mttkrp_sparse(self.ctx._ctx, C.byref(vB), C.byref(vC),
                                                     C.byref(vD), C.byref(opts), C.byref(r),
                                                     C.byref(st)))
            self.out_bytes = 8 * (r.nrows + 1) + 16 * r.nnz
            self.nnz_out = r.nnz
            self._sparse_mults = st.mults
        self.release(r)
        return st

    def post_step(self, r):
        """Dense result at N > 1: the cut slices' partial rows are completed
        by one all-gather (sharding.exchange_boundary_rows), in the step."""
        if not self.dist_on or self.spans is None:
            return
        from paper_1802_10574_b200 import sharding as S
        from paper_1802_10574_b200.kernels import _dev_tensor

        n = r.nrows * r.ncols
        if n == 0:
            return
        t = _dev_tensor(r.vals, n, "float64", None).view(r.nrows, r.ncols)
        S.exchange_boundary_rows(t, self.spans, "cuda")

    def step(self, timing=False):
        return self._call(self.vB, self.vC, self.vD, self.N.STAM_MEM_DEVICE, timing)

    def e2e_step(self):
        return self._call(self.hB, self.hC, self.hD, self.N.STAM_MEM_HOST, False)

    def local_flops(self):
        if self.useful is not None:
            return self.useful
        return 2 * getattr(self, "_sparse_mults", 0)

    def h2d_bytes(self):
        return self.own_in_bytes + self.shared_bytes

    def d2h_bytes(self):
        return self.out_bytes

    def total_units(self):
        return self.cfg["B"].dims[0]

    def ref_sample(self, slices):
        from paper_1802_10574_b200.storage import CSF3

        B = self.cfg["B"]
        f = int(B.pos1[slices])
        z = int(B.pos2[f])
        return CSF3((slices, B.dims[1], B.dims[2]), B.pos1[: slices + 1], B.idx1[:f],
                    B.pos2[: f + 1], B.idx2[:z], B.vals[:z])

    def ref_run(self, sub, nthreads):
        import oracle

        cfg = self.cfg
        if isinstance(cfg["C"].vals, np.ndarray) and cfg["C"].vals.ndim == 2:
            oracle.ref_mttkrp_dense(sub, cfg["C"].vals, cfg["D"].vals, nthreads)
            R = cfg["C"].vals.shape[1]
            nbytes = _csf_bytes(sub) + 8 * (cfg["C"].vals.size + cfg["D"].vals.size) + \
                8 * sub.dims[0] * R
            return nbytes, 2 * R * (sub.nnz + sub.nfibers)
        out = oracle.ref_mttkrp_sparse(sub, cfg["C"], cfg["D"], nthreads)
        nbytes = _csf_bytes(sub) + _csr_bytes(cfg["C"]) + _csr_bytes(cfg["D"]) + \
            8 * (out["nrows"] + 1) + 16 * int(out["pos"][-1])
        return nbytes, 0


WORKLOADS = {1: SpgemmWork, 2: SpaddWork, 3: SpgemmWork, 4: MttkrpWork, 5: MttkrpWork}


class FileSpgemmWork(SpgemmWork):
    """C = A*A for a Matrix Market file (SuiteSparse-style input; --mtx)."""

    def __init__(self, path: str):
        from paper_1802_10574_b200 import io as sio

        self.cid = 0
        self.name = f"file:{Path(path).name}:AxA"
        self.broadcast_ms, self.broadcast_bytes = 0.0, 0
        t = time.time()
        A = sio.load_matrix_market(path)
        if A.nrows != A.ncols:
            raise SystemExit("--mtx: A*A needs a square matrix")
        self.cfg = {"kind": "spgemm", "A": A, "B": A}
        self.gen_s = time.time() - t


class FileMttkrpWork(MttkrpWork):
    """Dense-factor MTTKRP on a FROSTT .tns file (order 3; --tns), seeded
    random factors of rank --rank."""

    def __init__(self, path: str, rank: int):
        from paper_1802_10574_b200 import generators as G
        from paper_1802_10574_b200 import io as sio

        self.cid = 0
        self.name = f"file:{Path(path).name}:R{rank}"
        self.broadcast_ms, self.broadcast_bytes = 0.0, 0
        t = time.time()
        B = sio.load_tns(path)
        if not hasattr(B, "pos1"):
            raise SystemExit("--tns: an order-3 tensor is needed")
        self.cfg = {"kind": "mttkrp_dense", "B": B, "C": G.dense(B.dims[1], rank, 401),
                    "D": G.dense(B.dims[2], rank, 402)}
        self.gen_s = time.time() - t


# ---------------------------------------------------------------------------
# clocks sampler
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, t0, t1):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [l for (t, l) in self.lines if t0 - 0.06 <= t <= t1 + 0.06] or [
            l for (_, l) in self.lines[-3:]]
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in rows:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except Exception:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference CPU path
# ---------------------------------------------------------------------------
def _ref_kind():
    import oracle

    if not oracle.ref_available():
        raise SystemExit("oracle/_ref missing; run __graft_entry__.build() where /root/reference "
                         "exists")
    return "reference"


def ref_timed(W, nthreads, target_s, reps=5):
    """The reference CPU path on a bounded sample of W's rows/slices: one
    discarded warm-up, then the median of `reps` timed runs.
    Returns (GB/s, useful GFLOP/s, units, seconds per run)."""
    units = W.total_units()
    t = time.perf_counter()
    probe = max(1, units // 200)
    W.ref_run(W.ref_sample(probe), nthreads)
    per_unit = (time.perf_counter() - t) / probe
    n = int(min(units, max(1, target_s / max(per_unit, 1e-9))))
    sample = W.ref_sample(n)
    W.ref_run(sample, nthreads)  # warm-up, discarded
    times = []
    nbytes = flops = 0
    for _ in range(reps):
        t = time.perf_counter()
        nbytes, flops = W.ref_run(sample, nthreads)
        times.append(time.perf_counter() - t)
    med = statistics.median(times)
    return nbytes / med / 1e9, flops / med / 1e9, n, med


def cpu_baselines(W, target_s):
    kind = _ref_kind()
    out = {}
    cores = os.cpu_count() or 1
    unit = "slices" if W.cid in (4, 5) else "rows"
    for label, nt in (("1thread", 1), ("all", cores)):
        v, g, n, med = ref_timed(W, nt, target_s)
        out[label] = {"value": v, "unit": "GB/s", "useful_gflops": g or None, "cores": nt,
                      "kind": kind,
                      "sample": f"first {n} of {W.total_units()} {unit}, median of 5 runs "
                                f"({med:.2f} s each) after a discarded warm-up; reference "
                                f"Workspace/TensorBuilder, {nt} thread(s)"
                                + (" (row blocks, one Workspace each)" if nt > 1 else "")}
    return out


def run_reference(args, cid):
    """--impl reference: the reference CPU path alone, rank 0 only, all host
    threads, each step a bounded sample of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    kind = _ref_kind()
    W = WORKLOADS[cid](cid)
    nthreads = os.cpu_count() or 1
    budget = 120.0 / max(1, args.steps + args.warmup)
    units = W.total_units()
    t = time.perf_counter()
    probe = max(1, units // 200)
    W.ref_run(W.ref_sample(probe), nthreads)
    per_unit = (time.perf_counter() - t) / probe
    n = int(min(units, max(1, budget / max(per_unit, 1e-9))))
    sample = W.ref_sample(n)
    for _ in range(args.warmup):
        W.ref_run(sample, nthreads)
    times, nbytes, flops = [], 0, 0
    for _ in range(args.steps):
        t = time.perf_counter()
        nbytes, flops = W.ref_run(sample, nthreads)
        times.append(time.perf_counter() - t)
    tot = sum(times)
    value = nbytes * args.steps / tot / 1e9
    unit = "slices" if cid in (4, 5) else "rows"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": W.name, "config_id": cid, "sample_units": n,
                   "total_units": units},
        "useful_gflops": (flops * args.steps / tot / 1e9) or None,
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": nthreads, "kind": kind,
                         "sample": f"first {n} of {units} {unit} per step, {nthreads} threads "
                                   f"(row blocks, one Workspace each)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    _emit(line)


# ---------------------------------------------------------------------------
# one config on this rank
# ---------------------------------------------------------------------------
def run_config(W, args, ctx, stream, world, rank, dist_on, local, cpu_target_s):
    import torch
    import torch.distributed as dist

    W.distribute(world, rank, dist_on)
    W.setup(ctx)
    flush = (torch.zeros(32 << 20, dtype=torch.float64, device="cuda")
             if (W.own_in_bytes + W.shared_bytes) <= L2_BYTES else None)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            W.step()
        torch.cuda.synchronize()
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()
        launches = 0
        if flush is None:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            t0 = time.time()
            ev0.record(stream)
            for _ in range(args.steps):
                st = W.step()
                launches += st.kernel_launches
            ev1.record(stream)
            torch.cuda.synchronize()
            t1 = time.time()
            ms = ev0.elapsed_time(ev1) / args.steps
        else:
            # inputs fit in L2: flush it before every step, time each step
            # with its own events (the flush is outside the timed region)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            t0 = time.time()
            for a, b in evs:
                flush.add_(1)
                a.record(stream)
                st = W.step()
                b.record(stream)
                launches += st.kernel_launches
            torch.cuda.synchronize()
            t1 = time.time()
            ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()
    clk = clocks.stop(t0, t1)
    # kernel timings (separate pass with per-kernel events recorded by the library)
    kms, tot_ms, kname = [], [], ""
    with torch.cuda.stream(stream):
        for _ in range(max(5, min(args.steps, 30))):
            if flush is not None:
                flush.add_(1)
            st = W.step(timing=True)
            kms.append(st.main_kernel_ms)
            tot_ms.append(st.total_kernel_ms)
            kname = st.main_kernel.decode()
    # e2e through the C ABI with pinned host buffers
    e2e_times = []
    for _ in range(max(3, min(args.steps, 8))):
        torch.cuda.synchronize()
        t = time.perf_counter()
        W.e2e_step()
        e2e_times.append(time.perf_counter() - t)
    e2e_s = statistics.median(e2e_times)

    algo = W.algo_bytes_total(dist_on)
    flops = float(W.local_flops())
    nnz_out = float(W.nnz_out)
    per_rank = torch.tensor([ms, e2e_s, -flops, -nnz_out, float(W.broadcast_ms)],
                            dtype=torch.float64, device="cuda")
    if dist_on:
        dist.all_reduce(per_rank, op=dist.ReduceOp.MAX)
        sums = torch.tensor([flops, nnz_out], dtype=torch.float64, device="cuda")
        dist.all_reduce(sums)
        flops, nnz_out = sums.tolist()
    ms_max, e2e_max, _, _, bcast_ms = per_rank.tolist()
    if rank != 0:
        return None
    peak, peak_src = _peak_hbm()
    # rank 0's own call: its algorithmic bytes over the device time of ALL its
    # kernels (single-kernel calls: that kernel); the dominant kernel is named
    # beside.  Calls that overlap kernels on two streams (SpGEMM) use the
    # smaller of the kernel-duration sum and the step time.
    own_algo = W.own_in_bytes + W.shared_bytes + W.out_bytes
    kernel_ms = statistics.mean(kms)
    total_kms = statistics.mean(tot_ms)
    overlapped = total_kms > ms
    basis_ms = min(total_kms, ms)
    achieved = own_algo / (basis_ms * 1e-3) / 1e9
    res = {
        "workload": W.name, "config_id": W.cid or None,
        "value": algo / (ms_max * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms_max,
        "useful_gflops": flops / (ms_max * 1e-3) / 1e9,
        "algo_bytes_per_step": algo, "nnz_out": int(nnz_out),
        "l2": "inputs larger than L2 (no flush)" if flush is None
              else "inputs smaller than L2: 256 MB L2 flush before every timed step",
        "kernel_ms": kernel_ms, "kernels_total_ms": total_kms,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _traffic(W.name, kname),
                     "kernel": kname, "kernel_share": kernel_ms / total_kms if total_kms else None,
                     "kernels_per_call": launches // max(1, args.steps),
                     "time_basis": ("device step time (the call's kernels overlap on two "
                                    "streams; their durations sum to %.3f ms)" % total_kms)
                     if overlapped else "sum of the call's kernel durations (CUDA events)",
                     "peak_source": peak_src,
                     **({"l2_gather": {"bytes_per_step": W.l2_gather,
                                       "achieved_gbs": W.l2_gather / (basis_ms * 1e-3) / 1e9,
                                       "note": "factor rows read per nonzero / fiber "
                                               "(L2-resident); the binding stream"}}
                        if getattr(W, "l2_gather", None) else {})},
        "e2e": {"value": algo / e2e_max / 1e9, "unit": "GB/s",
                "h2d_bytes_per_step": W.h2d_bytes(), "d2h_bytes_per_step": W.d2h_bytes(),
                "ms_per_step": e2e_max * 1e3},
        "gpu_launches": launches,
        "clocks": clk,
        "gen_s": W.gen_s,
    }
    if dist_on:
        res["broadcast"] = {"ms": bcast_ms, "bytes": W.broadcast_bytes,
                            "note": "shared operand broadcast once over NCCL before the steps "
                                    "(outside the timed step)"}
    if world == 1 and not args.no_cpu_baseline and W.cid:
        try:
            res["cpu_baselines"] = cpu_baselines(W, cpu_target_s)
        except SystemExit as e:
            res["cpu_baselines"] = {"error": str(e)}
        except Exception as e:  # the baseline must not kill the GPU number
            res["cpu_baselines"] = {"error": repr(e)}
    return res


# The contract is ONE JSON line on stdout.  Libraries print there too (NCCL
# writes its version banner to stdout when the communicator is created), so the
# process's stdout is pointed at stderr for the whole run and the line goes to
# a private duplicate of the original descriptor.
_OUT = None


def _capture_stdout():
    global _OUT
    if _OUT is None:
        sys.stdout.flush()
        _OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def _emit(line):
    out = _OUT if _OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    _capture_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=None,
                    help="one config (1..5) as the headline; default: all five, headline 5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=0.6,
                    help="target seconds per reference run in the cpu_baseline samples")
    ap.add_argument("--mtx", help="SpGEMM A*A on this Matrix Market file instead of a config")
    ap.add_argument("--tns", help="dense MTTKRP on this FROSTT .tns file instead of a config")
    ap.add_argument("--rank", type=int, default=32, help="factor rank for --tns")
    ap.add_argument("--mode", default="fused", choices=["fused", "assemble", "compute", "unsorted"],
                    help="execution mode (SpGEMM / SpAdd configs): SPEC.md:372-374, sort flag :351")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    headline = args.config or HEADLINE
    if headline not in WORKLOADS:
        raise SystemExit(f"config {headline} not available in this build")
    if args.impl == "reference":
        return run_reference(args, headline)

    import torch
    import torch.distributed as dist

    dist_on = "WORLD_SIZE" in os.environ and "RANK" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1")) if dist_on else 1
    rank = int(os.environ.get("RANK", "0")) if dist_on else 0
    local = int(os.environ.get("LOCAL_RANK", "0")) if dist_on else 0
    torch.cuda.set_device(local)
    if dist_on:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1802_10574_b200 import Context

    ctx = Context(local)
    stream = torch.cuda.Stream(device=local)
    ctx.set_stream(stream)

    if args.mtx or args.tns:
        cids = [0]
    elif args.config:
        cids = [args.config]
    else:
        cids = [c for c in (1, 2, 3, 4, 5) if c != headline] + [headline]
    results = {}
    for cid in cids:
        if cid == 0:
            W = FileSpgemmWork(args.mtx) if args.mtx else FileMttkrpWork(args.tns, args.rank)
        else:
            W = WORKLOADS[cid](cid, have_data=(rank == 0))
        if args.mode != "fused":
            if cid not in (0, 1, 2, 3) or args.tns:
                raise SystemExit("--mode applies to the SpGEMM and SpAdd configs (1, 2, 3)")
            W.mode = args.mode
        results[cid] = run_config(W, args, ctx, stream, world, rank, dist_on, local,
                                  args.cpu_seconds)
        del W
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    if rank == 0:
        h = results[cids[-1]]
        cb = h.get("cpu_baselines", {})
        line = {
            "metric": METRIC, "value": h["value"], "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": h["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64",
            "data": ("file " + (args.mtx or args.tns)) if cids[-1] == 0 else
                    "synthetic (seeded; BASELINE shapes, see DESIGN.md)",
            "config": {"workload": h["workload"], "config_id": h["config_id"],
                       "l2": h["l2"], "algo_bytes_per_step": h["algo_bytes_per_step"],
                       "nnz_out": h["nnz_out"],
                       **({"mode": args.mode} if args.mode != "fused" else {}),
                       "parallelism": f"row shards x{world} (strong)"},
            "useful_gflops": h["useful_gflops"],
            "kernel_ms": h["kernel_ms"], "kernels_total_ms": h["kernels_total_ms"],
            "roofline": h["roofline"],
            "e2e": h["e2e"],
            "gpu_launches": h["gpu_launches"],
            "clocks": h["clocks"],
        }
        if "broadcast" in h:
            line["broadcast"] = h["broadcast"]
        if "all" in cb:
            line["cpu_baseline"] = dict(cb["all"])
            line["cpu_baseline_1thread"] = cb["1thread"]
        elif cb:
            line["cpu_baseline"] = {"value": None, **cb}
        if len(cids) > 1:
            line["configs"] = {str(c): {k: v for k, v in r.items() if k != "clocks"}
                               for c, r in results.items()}
        _emit(line)
    if dist_on:
        dist.destroy_process_group()
    ctx.close()


if __name__ == "__main__":
    main()
