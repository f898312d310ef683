"""CPU: the oracle's SPEC kernels outside the workspace plans (TTV, row-dot,
merge-based SpAdd) against dense evaluation and the SPEC
properties (merge-based SpAdd: merge_compares >= nnz(B u C) - 1, workspace
SpAdd: merge_compares == 0)."""
import numpy as np
import pytest

import oracle
from paper_1802_10574_b200 import generators as G


def _dense(M):
    d = np.zeros((M.nrows, M.ncols))
    for i in range(M.nrows):
        for t in range(M.pos[i], M.pos[i + 1]):
            d[i, M.idx[t]] += M.vals[t]
    return d


def _from(out):
    d = np.zeros((out["nrows"], out["ncols"]))
    for i in range(out["nrows"]):
        for t in range(out["pos"][i], out["pos"][i + 1]):
            d[i, out["idx"][t]] = out["vals"][t]
    return d


@pytest.mark.parametrize("seed", range(4))
def test_rowdot_matches_dense(seed):
    B = G.csr_powerlaw(60, 50, seed, lmax=40)
    C = G.csr_powerlaw(60, 50, seed + 100, lmax=40)
    got = oracle.rowdot(B, C)["vals"]
    assert np.allclose(got, np.sum(_dense(B) * _dense(C), axis=1), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("k", [2, 3, 5])
def test_spadd_merge_matches_dense_and_counts(k):
    ops = [G.csr_powerlaw(80, 64, 10 + p, lmax=50) for p in range(k)]
    got = oracle.spadd_merge(ops)
    c = oracle.last_counters()
    want = sum(_dense(o) for o in ops)
    assert np.allclose(_from(got), want, rtol=1e-12, atol=1e-14)
    ws = oracle.spadd(ops)
    assert np.array_equal(got["pos"], ws["pos"]) and np.array_equal(got["idx"], ws["idx"])
    if k == 2:
        union = int(got["pos"][-1])
        assert c["merge_compares"] >= union - 1
    oracle.spadd(ops)
    assert oracle.last_counters()["merge_compares"] == 0


def test_ttv_matches_dense():
    B = G.csf3((12, 15, 20), G.slice_sizes_ranksize(12, 600, 1.5, 2), 3)
    c = np.random.default_rng(1).random(20)
    out = oracle.ttv(B, c)
    dense = np.zeros((12, 15))
    for i in range(12):
        for f in range(B.pos1[i], B.pos1[i + 1]):
            for p in range(B.pos2[f], B.pos2[f + 1]):
                dense[i, B.idx1[f]] += B.vals[p] * c[B.idx2[p]]
    assert np.allclose(_from(out), dense, rtol=1e-12, atol=1e-14)
    assert np.array_equal(out["pos"], B.pos1)
