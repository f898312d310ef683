"""GPU parity for the SPEC kernels outside the workspace plans:
TTV, row-dot and the merge-based SpAdd baseline vs the CPU oracle — values
bit-identical (sequential sums in coordinate order), structure identical,
merge_compares equal to the oracle's two-pointer loop count."""
import numpy as np
import pytest

import oracle
from paper_1802_10574_b200 import Dense
from paper_1802_10574_b200 import _native as N
from paper_1802_10574_b200 import generators as G

pytestmark = pytest.mark.gpu


def _np(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


@pytest.mark.parametrize("scale", [0.01, 0.05])
def test_ttv_config4_shape(ctx, scale):
    cfg = G.make_config(4, scale=scale)
    B = cfg["B"]
    c = G.dense(B.dims[2], 1, 9).vals.reshape(-1)
    got = ctx.ttv(B.to("cuda"), c)
    ref = oracle.ttv(B, c)
    oracle.compare_csr(got, ref, exact_values=True)


@pytest.mark.parametrize("seed", [0, 1])
def test_rowdot_bit_identical_and_counts(ctx, seed):
    B = G.csr_powerlaw(20000, 3000, seed, lmax=400)
    C = G.csr_powerlaw(20000, 3000, seed + 50, lmax=400)
    st = N.Stats()
    a = _np(ctx.rowdot(B.to("cuda"), C.to("cuda"), stats=st).vals).reshape(-1)
    ref = oracle.rowdot(B, C)
    cnt = oracle.last_counters()
    assert np.array_equal(a.view(np.int64), ref["vals"].view(np.int64))
    assert st.merge_compares == cnt["merge_compares"]
    assert st.mults == cnt["mults"]


@pytest.mark.parametrize("k", [2, 3, 6])
def test_spadd_merge_bit_identical_and_counts(ctx, k):
    ops = [G.csr_powerlaw(5000, 4000, 70 + p, lmax=300) for p in range(k)]
    st = N.Stats()
    D = ctx.spadd_merge([o.to("cuda") for o in ops], stats=st)
    ref = oracle.spadd_merge(ops)
    cnt = oracle.last_counters()
    oracle.compare_csr(D, ref, exact_values=True)
    assert st.merge_compares == cnt["merge_compares"]
    assert st.adds == cnt["adds"]
    ws = N.Stats()
    ctx.spadd([o.to("cuda") for o in ops], stats=ws)
    assert ws.merge_compares == 0  # the workspace plan has no merge


def test_spadd_merge_empty_rows(ctx):
    rng = np.random.default_rng(3)
    ops = []
    for p in range(3):
        lens = rng.integers(0, 5, size=300)
        lens[rng.random(300) < 0.5] = 0
        pos = np.zeros(301, dtype=np.int64)
        np.cumsum(lens, out=pos[1:])
        ops.append(G.csr_from_lengths(300, 10, pos, 90 + p))
    oracle.compare_csr(ctx.spadd_merge(ops), oracle.spadd_merge(ops), exact_values=True)
