"""Generates tests/golden/*.npz: seeded inputs and the outputs of the
REFERENCE's own stam::Workspace / stam::TensorBuilder (oracle/_ref, compiled
from /root/reference/proj/src by oracle/Makefile) driving the hot-path loop
nests.  The reference ships no golden vectors for this path (SURVEY §8c:
test_engine.cpp / test_oracle.cpp are one-line stubs, tests/golden absent), so
these fixtures pin the C restatement (oracle/stam_oracle.c) and the GPU kernels
to the reference's workspace semantics.

    python tests/golden/make_golden.py        # needs /root/reference
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_1802_10574_b200 import CSF3, CSR  # noqa: E402
from paper_1802_10574_b200 import generators as G  # noqa: E402

OUT = Path(__file__).resolve().parent


def save_csr(d, prefix, m):
    d[prefix + "_nrows"] = np.int64(m.nrows)
    d[prefix + "_ncols"] = np.int64(m.ncols)
    d[prefix + "_pos"], d[prefix + "_idx"], d[prefix + "_vals"] = m.pos, m.idx, m.vals


def save_csf(d, prefix, b):
    d[prefix + "_dims"] = np.array(b.dims, dtype=np.int64)
    for k in ("pos1", "idx1", "pos2", "idx2", "vals"):
        d[f"{prefix}_{k}"] = getattr(b, k)


def save_out(d, out):
    for k in ("pos", "idx", "vals"):
        if k in out:
            d["out_" + k] = out[k]


def main():
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref missing: build it with `make -C oracle` where /root/reference exists")
    cases = {}
    # SpGEMM: config-1 shape (scaled), config-3 power-law shape (scaled), SPEC examples
    cfg = G.make_config(1, scale=0.01)
    cases["spgemm_cfg1"] = ("spgemm", cfg["A"], cfg["B"])
    cfg = G.make_config(3, scale=0.0005)
    cases["spgemm_cfg3"] = ("spgemm", cfg["A"], cfg["A"])
    n = 16
    eye = CSR(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.ones(n))
    cases["spgemm_identity"] = ("spgemm", eye, eye)
    rng = np.random.default_rng(40)
    a = np.round(rng.random((40, 40)) * (rng.random((40, 40)) < 0.1), 6)
    b = np.round(rng.random((40, 40)) * (rng.random((40, 40)) < 0.1), 6)
    cases["spgemm_40x40"] = ("spgemm", CSR.from_dense(a), CSR.from_dense(b))
    # SpAdd: config-2 shape (scaled), overlapping narrow operands
    cfg = G.make_config(2, scale=0.0005)
    cases["spadd_cfg2"] = ("spadd", *cfg["ops"])
    cases["spadd_overlap"] = ("spadd", *[G.csr_fixed(60, 40, 12, 700 + k) for k in range(4)])
    # MTTKRP dense and sparse (scaled config shapes)
    cfg = G.make_config(4, scale=0.002)
    cases["mttkrp_dense_cfg4"] = ("mttkrp_dense", cfg["B"], cfg["C"].vals, cfg["D"].vals)
    cfg = G.make_config(5, scale=0.0002)
    cases["mttkrp_sparse_cfg5"] = ("mttkrp_sparse", cfg["B"], cfg["C"], cfg["D"])
    sizes = np.full(12, 80, dtype=np.int64)
    Bm = G.csf3((12, 10, 20), sizes, 77)
    cases["mttkrp_sparse_multi"] = ("mttkrp_sparse", Bm, G.csr_fixed(10, 48, 20, 78),
                                    G.csr_fixed(20, 48, 15, 79))

    for name, (kind, *args) in cases.items():
        d = {"kind": np.array(kind)}
        if kind == "spgemm":
            save_csr(d, "A", args[0])
            save_csr(d, "B", args[1])
            out = oracle.ref_spgemm(args[0], args[1])
        elif kind == "spadd":
            d["nops"] = np.int64(len(args))
            for k, m in enumerate(args):
                save_csr(d, f"op{k}", m)
            out = oracle.ref_spadd(list(args))
        elif kind == "mttkrp_dense":
            save_csf(d, "B", args[0])
            d["C"], d["D"] = args[1], args[2]
            out = oracle.ref_mttkrp_dense(args[0], args[1], args[2])
        else:
            save_csf(d, "B", args[0])
            save_csr(d, "C", args[1])
            save_csr(d, "D", args[2])
            out = oracle.ref_mttkrp_sparse(args[0], args[1], args[2])
        save_out(d, out)
        np.savez_compressed(OUT / f"{name}.npz", **d)
        print(name, {k: v.shape for k, v in d.items() if hasattr(v, "shape") and v.ndim})


if __name__ == "__main__":
    main()
