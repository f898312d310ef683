"""Loads tests/golden/*.npz fixtures (inputs + reference outputs)."""
from pathlib import Path

import numpy as np

from paper_1802_10574_b200 import CSF3, CSR, Dense

GOLDEN = Path(__file__).resolve().parent / "golden"


def names():
    return sorted(p.stem for p in GOLDEN.glob("*.npz"))


def _csr(d, p):
    return CSR(int(d[p + "_nrows"]), int(d[p + "_ncols"]), d[p + "_pos"], d[p + "_idx"],
               d[p + "_vals"])


def _csf(d, p):
    return CSF3(tuple(int(x) for x in d[p + "_dims"]), d[p + "_pos1"], d[p + "_idx1"],
                d[p + "_pos2"], d[p + "_idx2"], d[p + "_vals"])


def load(name):
    d = dict(np.load(GOLDEN / f"{name}.npz"))
    kind = str(d["kind"])
    if kind == "spgemm":
        args = (_csr(d, "A"), _csr(d, "B"))
    elif kind == "spadd":
        args = ([_csr(d, f"op{k}") for k in range(int(d["nops"]))],)
    elif kind == "mttkrp_dense":
        args = (_csf(d, "B"), Dense(d["C"]), Dense(d["D"]))
    else:
        args = (_csf(d, "B"), _csr(d, "C"), _csr(d, "D"))
    out = {k[4:]: v for k, v in d.items() if k.startswith("out_")}
    return kind, args, out
