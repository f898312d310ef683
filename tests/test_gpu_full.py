"""GPU parity at BASELINE's full sizes (configs 3 and 5 against the oracle,
all configs through size-independent properties).

* Oracle comparisons: structure bit-exact, values within the scaled bound
  |x - x_ref| <= 1e-12 * max(|x_ref|, sum|terms|); the oracle runs
  row-block threaded on the host's cores.
* Properties (checkers only, scipy on the host): linearity of every loop nest
  in a random vector x — C x = A (B x) for SpGEMM, D x = sum_q ops_q x for
  SpAdd — with the bound PTOL * (|A| (|B| |x|)) computed on absolute values
  (a checksum of checksums
  that does not depend on the accumulation order the GPU uses).  PTOL = 1e-10:
  the products x and the scipy evaluation add their own rounding (rows of up
  to 9e4 terms, n * eps ~ 1e-11 in the worst case); value parity itself is the
  oracle comparison's 1e-12 scaled bound.  (Config 4's and config 2's full-size oracle
  comparisons are in tests/test_gpu_mttkrp.py and tests/test_gpu_spadd.py.)
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from paper_1802_10574_b200 import generators as G

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

PTOL = 1e-10


def _d(x):
    return x.to("cuda")


def _sp(m):
    return sp.csr_matrix((np.asarray(m.vals), np.asarray(m.idx), np.asarray(m.pos)),
                         shape=(m.nrows, m.ncols))


def _abs(m):
    a = m.copy()
    a.data = np.abs(a.data)
    return a


def test_spgemm_config3_full_oracle(ctx):
    cfg = G.make_config(3)
    C = ctx.spgemm(_d(cfg["A"]), _d(cfg["B"]), result="host")
    rep = oracle.compare_csr(C, oracle.spgemm(cfg["A"], cfg["B"], nthreads=oracle.threads_default()))
    assert rep["nnz"] > 250_000_000


def test_mttkrp_sparse_config5_full_oracle(ctx):
    cfg = G.make_config(5)
    A = ctx.mttkrp(_d(cfg["B"]), _d(cfg["C"]), _d(cfg["D"]), result="host")
    rep = oracle.compare_csr(A, oracle.mttkrp_sparse(cfg["B"], cfg["C"], cfg["D"],
                                                     oracle.threads_default()))
    assert rep["nnz"] > 40_000_000


@pytest.mark.parametrize("cid", [1, 3])
def test_spgemm_full_linearity(ctx, cid):
    cfg = G.make_config(cid)
    C = _sp(ctx.spgemm(_d(cfg["A"]), _d(cfg["B"]), result="host"))
    A, B = _sp(cfg["A"]), _sp(cfg["B"])
    x = np.random.default_rng(cid).uniform(-1, 1, B.shape[1])
    got, ref = C @ x, A @ (B @ x)
    bound = PTOL * (_abs(A) @ (_abs(B) @ np.abs(x)))
    assert np.all(np.abs(got - ref) <= bound + 1e-300)


def test_spadd_config2_full_linearity(ctx):
    cfg = G.make_config(2)
    ops = cfg["ops"]
    D = _sp(ctx.spadd([_d(o) for o in ops], result="host"))
    x = np.random.default_rng(2).uniform(-1, 1, D.shape[1])
    S = [_sp(o) for o in ops]
    ref = sum(s @ x for s in S)
    bound = PTOL * sum(_abs(s) @ np.abs(x) for s in S)
    assert np.all(np.abs(D @ x - ref) <= bound + 1e-300)
    # union structure: every operand entry is present in D
    for s in S:
        assert (abs(s).astype(bool) > D.astype(bool)).nnz == 0
