#!/usr/bin/env python
"""Benchmark of the hot path.

One "step" = one call of the kernel entry point (C ABI) over one batch of
synthetic input with BASELINE.json's shapes.  Default workload: BASELINE
configs[1] (config 2, SpAdd D = A+B+C, 3 x 200k x 200k, 50/row); ``--config``
selects any of the five.

Our arm (default):
  value    = algorithmic HBM bytes of the call (inputs read once + output written
             once, int64 indices / fp64 values) / device time per step, with the
             inputs resident in HBM; whole-job aggregate over ranks.
  e2e      = the same metric through the same C-ABI call with pinned HOST
             inputs and a HOST result (H2D + D2H inside the timed region).
  roofline = dominant kernel's algorithmic bytes / its CUDA-event duration vs
             the measured HBM copy bandwidth (MEASURED_PEAKS.json).
  cpu_baseline = the reference CPU path (oracle/_ref: the reference's own
             Workspace/TensorBuilder) on the host cores, bounded sample.

``--impl reference``: rank 0 times the reference CPU path alone on the same
config/metric (other ranks exit), printing the same JSON line.

Multi-GPU (torchrun): weak scaling — every rank processes its own full-size
shard of the row (slice) dimension with independently seeded inputs; no
collective on the data path; time = max over ranks.
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


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def _csr_bytes(m) -> int:
    return 8 * (m.nrows + 1) + 16 * m.nnz


def _csf_bytes(b) -> int:
    return 8 * (b.dims[0] + 1) + 8 * b.nfibers + 8 * (b.nfibers + 1) + 16 * b.nnz


class Workload:
    """Common driver: inputs on device, raw C-ABI step, e2e step, CPU ref."""

    mode = "fused"  # fused | assemble | compute | unsorted (SpGEMM, SpAdd)

    def __init__(self, cid: int, shard: int):
        from paper_1802_10574_b200 import generators as G

        self.cid = cid
        self.name = G.CONFIG_NAMES[cid]
        t = time.time()
        self.cfg = G.make_config(cid, shard=shard)
        self.gen_s = time.time() - t

    # populated by subclasses
    def setup(self, ctx):
        raise NotImplementedError

    def step(self, timing=False):
        raise NotImplementedError

    def e2e_step(self):
        raise NotImplementedError


class SpaddWork(Workload):
    def setup(self, ctx):
        from paper_1802_10574_b200 import _native as N

        self.N = N
        self.ctx = ctx
        self.lib = N.load()
        self.dev = [o.to("cuda") for o in self.cfg["ops"]]
        self.views = (N.CsrView * len(self.dev))(*[o.view() for o in self.dev])
        import torch

        self.pinned = []
        for o in self.cfg["ops"]:
            arrs = [torch.from_numpy(a).pin_memory() for a in (o.pos, o.idx, o.vals)]
            self.pinned.append(arrs)
        from paper_1802_10574_b200.storage import CSR

        hops = [CSR(o.nrows, o.ncols, *arrs) for o, arrs in zip(self.cfg["ops"], self.pinned)]
        self.hviews = (N.CsrView * len(hops))(*[h.view() for h in hops])
        for v in self.hviews:
            v.mem = N.STAM_MEM_HOST
        self.in_bytes = sum(_csr_bytes(o) for o in self.cfg["ops"])
        self.nnz_out = None

    def _index(self, views):
        """Pre-assembled index for compute mode (assembled once, reused)."""
        if getattr(self, "_idx", None) is None:
            N = self.N
            r = N.CsrResult()
            opts = N.Options(1, N.STAM_MODE_ASSEMBLE, N.STAM_MEM_DEVICE, 0)
            N.check(self.lib.stam_cuda_spadd(self.ctx._ctx, len(self.dev), self.views,
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
                self.ctx._ctx, len(self.dev), views, C.byref(self._index(views)), C.byref(opts),
                C.byref(r), C.byref(st)))
        else:
            N.check(self.lib.stam_cuda_spadd(self.ctx._ctx, len(self.dev), views, C.byref(opts),
                                             C.byref(r), C.byref(st)))
        nnz, nrows = r.nnz, r.nrows
        N.check(self.lib.stam_cuda_release(self.ctx._ctx, C.c_void_p(r.handle)))
        self.nnz_out = nnz
        self.out_bytes = 8 * (nrows + 1) + 16 * nnz
        return st

    def step(self, timing=False):
        return self._call(self.views, self.N.STAM_MEM_DEVICE, timing)

    def e2e_step(self):
        return self._call(self.hviews, self.N.STAM_MEM_HOST, False)

    def algo_bytes(self):
        return self.in_bytes + self.out_bytes

    def flops(self):
        # workspace adds executed (SPEC counters: every accumulate insert)
        return sum(o.nnz for o in self.cfg["ops"][1:])

    def h2d_bytes(self):
        return self.in_bytes

    def d2h_bytes(self):
        return self.out_bytes

    # reference CPU path on a row sample
    def ref_sample(self, rows):
        import numpy as np
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

    def total_rows(self):
        return self.cfg["ops"][0].nrows


class SpgemmWork(Workload):
    """C = A*B (configs 1 and 3; config 3 squares A, so B is A)."""

    def setup(self, ctx):
        from paper_1802_10574_b200 import _native as N
        from paper_1802_10574_b200.storage import CSR
        import torch

        self.N, self.ctx, self.lib = N, ctx, N.load()
        A, B = self.cfg["A"], self.cfg["B"]
        self.same = B is A
        self.Ad = A.to("cuda")
        self.Bd = self.Ad if self.same else B.to("cuda")
        self.va, self.vb = self.Ad.view(), self.Bd.view()
        pin = lambda m: CSR(m.nrows, m.ncols, *[torch.from_numpy(a).pin_memory()
                                                for a in (m.pos, m.idx, m.vals)])
        self.Ah = pin(A)
        self.Bh = self.Ah if self.same else pin(B)
        self.ha, self.hb = self.Ah.view(), self.Bh.view()
        self.in_bytes = _csr_bytes(A) + (0 if self.same else _csr_bytes(B))
        self.products = int(np.sum(np.diff(B.pos)[A.idx]))
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
        N.check(self.lib.stam_cuda_release(self.ctx._ctx, C.c_void_p(r.handle)))
        return st

    def step(self, timing=False):
        return self._call(self.va, self.vb, self.N.STAM_MEM_DEVICE, timing)

    def e2e_step(self):
        return self._call(self.ha, self.hb, self.N.STAM_MEM_HOST, False)

    def algo_bytes(self):
        return self.in_bytes + self.out_bytes

    def flops(self):
        return 2 * self.products

    def h2d_bytes(self):
        return self.in_bytes

    def d2h_bytes(self):
        return self.out_bytes

    def ref_sample(self, rows):
        from paper_1802_10574_b200.storage import CSR

        A = self.cfg["A"]
        e = int(A.pos[rows])
        return (CSR(rows, A.ncols, A.pos[: rows + 1], A.idx[:e], A.vals[:e]), self.cfg["B"])

    def ref_run(self, sample, nthreads):
        import oracle

        A, B = sample
        out = oracle.ref_spgemm(A, B, nthreads)
        nbytes = _csr_bytes(A) + (0 if self.same else _csr_bytes(B)) + 8 * (out["nrows"] + 1) + \
            16 * int(out["pos"][-1])
        return nbytes, 2 * int(np.sum(np.diff(B.pos)[A.idx]))

    def total_rows(self):
        return self.cfg["A"].nrows


class MttkrpWork(Workload):
    """A = B x_2 C x_3 D: dense factors (config 4) or CSR factors (config 5)."""

    def setup(self, ctx):
        from paper_1802_10574_b200 import _native as N
        from paper_1802_10574_b200.storage import CSF3, CSR, Dense
        import torch

        self.N, self.ctx, self.lib = N, ctx, N.load()
        B, Cf, Df = self.cfg["B"], self.cfg["C"], self.cfg["D"]
        self.dense = isinstance(Cf, Dense)
        self.Bd, self.Cd, self.Dd = B.to("cuda"), Cf.to("cuda"), Df.to("cuda")
        self.vB, self.vC, self.vD = self.Bd.view(), self.Cd.view(), self.Dd.view()
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        self.Bh = CSF3(B.dims, *[pin(a) for a in (B.pos1, B.idx1, B.pos2, B.idx2, B.vals)])
        if self.dense:
            self.Ch, self.Dh = Dense(pin(Cf.vals)), Dense(pin(Df.vals))
            self.in_bytes = _csf_bytes(B) + 8 * (Cf.vals.size + Df.vals.size)
            self.R = Cf.ncols
            self.useful = 2 * self.R * (B.nnz + B.nfibers)
            # every nonzero reads a factor row of D and every fiber one of C:
            # the loop nest's operand stream from L2
            self.l2_gather = 8 * self.R * (B.nnz + B.nfibers)
        else:
            self.Ch = CSR(Cf.nrows, Cf.ncols, *[pin(a) for a in (Cf.pos, Cf.idx, Cf.vals)])
            self.Dh = CSR(Df.nrows, Df.ncols, *[pin(a) for a in (Df.pos, Df.idx, Df.vals)])
            self.in_bytes = _csf_bytes(B) + _csr_bytes(Cf) + _csr_bytes(Df)
            self.R = Cf.ncols
            self.useful = None
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
        else:
            r = N.CsrResult()
            N.check(self.lib.stam_cuda_mttkrp_sparse(self.ctx._ctx, C.byref(vB), C.byref(vC),
                                                     C.byref(vD), C.byref(opts), C.byref(r),
                                                     C.byref(st)))
            self.out_bytes = 8 * (r.nrows + 1) + 16 * r.nnz
            self.nnz_out = r.nnz
            self._sparse_mults = st.mults
        N.check(self.lib.stam_cuda_release(self.ctx._ctx, C.c_void_p(r.handle)))
        return st

    def step(self, timing=False):
        return self._call(self.vB, self.vC, self.vD, self.N.STAM_MEM_DEVICE, timing)

    def e2e_step(self):
        return self._call(self.hB, self.hC, self.hD, self.N.STAM_MEM_HOST, False)

    def algo_bytes(self):
        return self.in_bytes + self.out_bytes

    def flops(self):
        if self.useful is not None:
            return self.useful
        return 2 * getattr(self, "_sparse_mults", 0)

    def h2d_bytes(self):
        return self.in_bytes

    def d2h_bytes(self):
        return self.out_bytes

    def ref_sample(self, slices):
        from paper_1802_10574_b200.storage import CSF3

        B = self.cfg["B"]
        f = int(B.pos1[slices])
        z = int(B.pos2[f])
        sub = CSF3((slices, B.dims[1], B.dims[2]), B.pos1[: slices + 1], B.idx1[:f],
                   B.pos2[: f + 1], B.idx2[:z], B.vals[:z])
        return sub

    def ref_run(self, sub, nthreads):
        import oracle

        if self.dense:
            oracle.ref_mttkrp_dense(sub, self.cfg["C"].vals, self.cfg["D"].vals, nthreads)
            nbytes = _csf_bytes(sub) + 8 * (self.cfg["C"].vals.size + self.cfg["D"].vals.size) + \
                8 * sub.dims[0] * self.R
            return nbytes, 2 * self.R * (sub.nnz + sub.nfibers)
        out = oracle.ref_mttkrp_sparse(sub, self.cfg["C"], self.cfg["D"], nthreads)
        nbytes = _csf_bytes(sub) + _csr_bytes(self.cfg["C"]) + _csr_bytes(self.cfg["D"]) + \
            8 * (out["nrows"] + 1) + 16 * int(out["pos"][-1])
        return nbytes, 0

    def total_rows(self):
        return self.cfg["B"].dims[0]


WORKLOADS = {1: SpgemmWork, 2: SpaddWork, 3: SpgemmWork, 4: MttkrpWork, 5: MttkrpWork}


class FileSpgemmWork(SpgemmWork):
    """C = A*A for a Matrix Market file (SuiteSparse-style input; --mtx)."""

    def __init__(self, path: str):
        from paper_1802_10574_b200 import io as sio

        self.cid = 0
        self.name = f"file:{Path(path).name}:AxA"
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

    def mark(self):
        return time.time()

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
def run_reference(args, cid):
    """--impl reference: the reference CPU path alone, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    W = WORKLOADS[cid](cid, 0)
    kind = "reference" if oracle.ref_available() else "port"
    if kind != "reference":
        raise SystemExit("oracle/_ref missing; run __graft_entry__.build() where /root/reference exists")
    nthreads = os.cpu_count() or 1
    rows = W.total_rows()
    # size the per-step sample so the whole run ends within a few minutes
    t = time.perf_counter()
    W.ref_run(W.ref_sample(max(1, rows // 20)), nthreads)
    est_full = (time.perf_counter() - t) * 20
    budget = 150.0 / max(1, args.steps + args.warmup)
    if est_full > budget:
        rows = max(1, int(rows * budget / est_full))
    sample = W.ref_sample(rows)
    for _ in range(args.warmup):
        W.ref_run(sample, nthreads)
    times, nbytes, flops = [], 0, 0
    for _ in range(args.steps):
        t = time.perf_counter()
        nbytes, flops = W.ref_run(sample, nthreads)
        times.append(time.perf_counter() - t)
    tot = sum(times)
    value = nbytes * args.steps / tot / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": W.name, "config_id": cid, "sample_rows": rows,
                   "total_rows": W.total_rows()},
        "useful_gflops": flops * args.steps / tot / 1e9,
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": nthreads, "kind": kind,
                         "sample": f"first {rows} of {W.total_rows()} rows per step, "
                                   f"{nthreads} threads (row blocks, one Workspace each)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(W, target_s=10.0):
    import oracle

    kind = "reference" if oracle.ref_available() else "port"
    nthreads = os.cpu_count() or 1
    rows = W.total_rows()
    sample = W.ref_sample(rows)
    reps, t_all, nbytes = 0, 0.0, 0
    rates = []
    while (t_all < target_s and reps < 5) or reps < 2:
        t = time.perf_counter()
        if kind == "reference":
            nbytes, _ = W.ref_run(sample, nthreads)
        dt = time.perf_counter() - t
        rates.append(nbytes / dt / 1e9)
        t_all += dt
        reps += 1
    return {"value": statistics.median(rates), "unit": "GB/s", "cores": nthreads, "kind": kind,
            "sample": f"full config, {reps} repetitions, median; reference Workspace/"
                      f"TensorBuilder over {nthreads} host threads (row blocks)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mtx", help="SpGEMM A*A on this Matrix Market file instead of a config")
    ap.add_argument("--tns", help="dense MTTKRP on this FROSTT .tns file instead of a config")
    ap.add_argument("--rank", type=int, default=32, help="factor rank for --tns")
    ap.add_argument("--mode", default="fused", choices=["fused", "assemble", "compute", "unsorted"],
                    help="execution mode (SpGEMM / SpAdd configs): SPEC.md:372-374, sort flag :351")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cid = args.config
    if cid not in WORKLOADS:
        raise SystemExit(f"config {cid} not available in this build")
    if args.impl == "reference":
        return run_reference(args, cid)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1802_10574_b200 import Context

    if args.mtx:
        W = FileSpgemmWork(args.mtx)
    elif args.tns:
        W = FileMttkrpWork(args.tns, args.rank)
    else:
        W = WORKLOADS[cid](cid, rank)
    if args.mode != "fused":
        if cid not in (1, 2, 3) and not args.mtx:
            raise SystemExit("--mode applies to the SpGEMM and SpAdd configs (1, 2, 3)")
        W.mode = args.mode
    ctx = Context(local)
    stream = torch.cuda.Stream(device=local)
    ctx.set_stream(stream)
    W.setup(ctx)

    # L2 is 126 MB: workloads whose inputs fit are timed with a flush (a
    # 256 MB read-modify-write) before every step
    flush = (torch.zeros(32 << 20, dtype=torch.float64, device="cuda")
             if W.in_bytes <= L2_BYTES else None)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            W.step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        launches = 0
        if flush is None:
            t0 = time.time()
            ev0.record(stream)
            for _ in range(args.steps):
                st = W.step()
                launches += st.kernel_launches
            ev1.record(stream)
            torch.cuda.synchronize()
            t1 = time.time()
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
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    clk = clocks.stop(t0, t1)
    if flush is None:
        ms = ev0.elapsed_time(ev1) / args.steps
    else:
        ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    # kernel timings (separate pass with per-kernel events)
    kms, tot_ms, kname = [], [], ""
    with torch.cuda.stream(stream):
        for _ in range(max(5, min(args.steps, 50))):
            if flush is not None:
                flush.add_(1)
            st = W.step(timing=True)
            kms.append(st.main_kernel_ms)
            tot_ms.append(st.total_kernel_ms)
            kname = st.main_kernel.decode()
    kernel_ms = statistics.mean(kms)
    # e2e through the C ABI with pinned host buffers
    e2e_times = []
    for _ in range(max(3, min(args.steps, 10))):
        torch.cuda.synchronize()
        t = time.perf_counter()
        W.e2e_step()
        e2e_times.append(time.perf_counter() - t)
    e2e_s = statistics.median(e2e_times)

    algo = W.algo_bytes()
    per_rank = torch.tensor([ms, e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(per_rank, op=dist.ReduceOp.MAX)
    ms_max, e2e_max = per_rank.tolist()
    value = algo * world / (ms_max * 1e-3) / 1e9
    peak, peak_src = _peak_hbm()
    # the call's algorithmic bytes over the device time of ALL its kernels
    # (single-kernel calls: that kernel); the dominant kernel is named beside.
    # Calls that run kernels on two streams at once (SpGEMM) overlap them, so
    # the basis is the smaller of the kernel-duration sum and the step time.
    total_kms = statistics.mean(tot_ms)
    overlapped = total_kms > ms
    basis_ms = min(total_kms, ms)
    achieved = algo / (basis_ms * 1e-3) / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": ("file " + (args.mtx or args.tns)) if W.cid == 0 else
                    "synthetic (seeded; BASELINE shapes, see DESIGN.md)",
            "config": {"workload": W.name, "config_id": cid if W.cid else None,
                       "l2": "inputs larger than L2 (no flush)" if flush is None
                       else "inputs smaller than L2: 256 MB L2 flush before every timed step",
                       "algo_bytes_per_step": algo, "nnz_out": W.nnz_out,
                       **({"mode": W.mode} if W.mode != "fused" else {}),
                       "parallelism": f"row shards x{world} (weak)"},
            "useful_gflops": W.flops() * world / (ms_max * 1e-3) / 1e9,
            "kernel_ms": kernel_ms, "kernels_total_ms": statistics.mean(tot_ms),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _traffic(W.name, kname),
                         "kernel": kname, "kernel_share": kernel_ms / total_kms,
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
            "e2e": {"value": algo * world / e2e_max / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": W.h2d_bytes(), "d2h_bytes_per_step": W.d2h_bytes(),
                    "ms_per_step": e2e_max * 1e3},
            "gpu_launches": launches,
            "clocks": clk,
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline(W)
            except Exception as e:  # the baseline must not kill the GPU number
                line["cpu_baseline"] = {"value": None, "error": str(e)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    ctx.close()


if __name__ == "__main__":
    main()
