"""Paper sparse-result MTTKRP experiment (PAPER §6.4): the
sparse-factor plan (CSR C, D; presence-checked w0; CSR A) against the
dense-factor plan (dense C, D, dense A) as the factor density sweeps.
B: 3-order CSF, I = J = K = `dim`, `nnz` uniform nonzeros (config-5 law);
factors: rank R = 256 with round(density * R) distinct columns per row (the
dense plan gets the same factors densified).  CSV: density, plan, kernel_ms
(median of 5, sum of the call's kernels), nnz(A)."""
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1802_10574_b200 import Context, Dense, _native as N  # noqa: E402
from paper_1802_10574_b200 import generators as G  # noqa: E402

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
nnz = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000_000
R = 256
ctx = Context(0)
B = G.csf3((dim, dim, dim), G.slice_sizes_uniform(dim, nnz, 5), 11).to("cuda")


def dense_of(M):
    d = np.zeros((M.nrows, M.ncols))
    rows = np.repeat(np.arange(M.nrows), np.diff(M.pos))
    d[rows, M.idx] = M.vals
    return Dense(d).to("cuda")


def timed(fn):
    ts = []
    for rep in range(6):
        st = N.Stats()
        out = fn(st)
        if rep:
            ts.append(st.total_kernel_ms)
    return statistics.median(ts), out


print("density,plan,kernel_ms,nnz_A")
for per_row in (1, 2, 4, 8, 16, 32, 64, 128, 256):
    Cs = G.csr_fixed(dim, R, per_row, 21)
    Ds = G.csr_fixed(dim, R, per_row, 22)
    t_s, A_s = timed(lambda st: ctx.mttkrp(B, Cs.to("cuda"), Ds.to("cuda"), timing=True, stats=st))
    print(f"{per_row / R:.4f},sparse,{t_s:.3f},{A_s.nnz}", flush=True)
    Cd, Dd = dense_of(Cs), dense_of(Ds)
    t_d, _ = timed(lambda st: ctx.mttkrp(B, Cd, Dd, timing=True, stats=st))
    print(f"{per_row / R:.4f},dense,{t_d:.3f},{dim * R}", flush=True)
    del A_s, Cd, Dd
