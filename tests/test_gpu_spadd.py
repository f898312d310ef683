"""GPU parity: SpAdd through the C ABI vs the CPU oracle (bit-exact).

The reference's SpAdd is the three-stage workspace sequence
``w0 = B; w0 += C; w0 += D`` (tests/test_transform.cpp:275-284) with a sorted
drain; the GPU rank-merge reproduces it exactly, so values are compared
bit-for-bit, structure by array equality."""
import numpy as np
import pytest

import oracle
from paper_1802_10574_b200 import CSR, StamError
from paper_1802_10574_b200 import generators as G

pytestmark = pytest.mark.gpu


def _dev(ops):
    return [o.to("cuda") for o in ops]


@pytest.mark.parametrize("scale", [0.001, 0.02, 0.2])
def test_spadd_config2_scaled(ctx, scale):
    cfg = G.make_config(2, scale=scale)
    D = ctx.spadd(_dev(cfg["ops"]))
    rep = oracle.compare_csr(D, oracle.spadd(cfg["ops"]), exact_values=True)
    assert rep["bit_identical"]


def test_spadd_config2_full(ctx):
    cfg = G.make_config(2)
    D = ctx.spadd(_dev(cfg["ops"]))
    ref = oracle.spadd(cfg["ops"], nthreads=oracle.threads_default())
    oracle.compare_csr(D, ref, exact_values=True)


def test_spadd_host_inputs_host_result(ctx):
    cfg = G.make_config(2, scale=0.01)
    D = ctx.spadd(cfg["ops"], result="host")
    assert isinstance(D.pos, np.ndarray)
    oracle.compare_csr(D, oracle.spadd(cfg["ops"]), exact_values=True)


@pytest.mark.parametrize("nops", [2, 3, 5, 16])
def test_spadd_many_operands_overlapping(ctx, nops):
    # narrow column range forces many coincident columns across operands
    ops = [G.csr_fixed(300, 64, 20, 900 + k) for k in range(nops)]
    D = ctx.spadd(_dev(ops))
    oracle.compare_csr(D, oracle.spadd(ops), exact_values=True)


def test_spadd_ragged_and_empty_rows(ctx):
    rng = np.random.default_rng(5)
    ops = []
    for k in range(3):
        lens = rng.integers(0, 40, size=500)
        lens[rng.random(500) < 0.3] = 0
        pos = np.zeros(501, dtype=np.int64)
        np.cumsum(lens, out=pos[1:])
        ops.append(G.csr_from_lengths(500, 1000, pos, 77 + k))
    D = ctx.spadd(_dev(ops))
    oracle.compare_csr(D, oracle.spadd(ops), exact_values=True)


def test_spadd_long_rows_take_the_bitmap_path(ctx):
    # rows far longer than a warp's staging buffer (384 entries) plus short rows
    rng = np.random.default_rng(9)
    ops = []
    for k in range(3):
        lens = rng.integers(1, 30, size=64)
        lens[[3, 17, 40]] = [5000, 150_000, 90_000]
        pos = np.zeros(65, dtype=np.int64)
        np.cumsum(lens, out=pos[1:])
        ops.append(G.csr_from_lengths(64, 200_000, pos, 31 + k))
    D = ctx.spadd(_dev(ops))
    oracle.compare_csr(D, oracle.spadd(ops), exact_values=True)


def test_spadd_postponed_rows(ctx):
    # two rows per warp whose sum exceeds the staging buffer but each fits
    pos = np.zeros(33, dtype=np.int64)
    lens = np.full(32, 120)
    np.cumsum(lens, out=pos[1:])
    ops = [G.csr_from_lengths(32, 100_000, pos, 61 + k) for k in range(3)]
    D = ctx.spadd(_dev(ops))
    oracle.compare_csr(D, oracle.spadd(ops), exact_values=True)


def test_spadd_all_empty(ctx):
    ops = [CSR(10, 10, np.zeros(11, np.int64), np.zeros(0, np.int64), np.zeros(0))
           for _ in range(3)]
    D = ctx.spadd(_dev(ops))
    assert D.nnz == 0 and np.array_equal(D.pos.cpu().numpy(), np.zeros(11))


def test_spadd_signed_zero_and_cancellation(ctx):
    # explicit zeros from cancellation are kept; -0.0 + 0.0 rules
    a = CSR(1, 4, np.array([0, 3]), np.array([0, 1, 2]), np.array([1.0, -0.0, 2.0]))
    b = CSR(1, 4, np.array([0, 3]), np.array([0, 1, 3]), np.array([-1.0, -0.0, -0.0]))
    for m in (a, b):
        m.pos, m.idx = m.pos.astype(np.int64), m.idx.astype(np.int64)
    D = ctx.spadd(_dev([a, b]))
    ref = oracle.spadd([a, b])
    oracle.compare_csr(D, ref, exact_values=True)
    assert list(ref["idx"]) == [0, 1, 2, 3]


def test_spadd_dimension_mismatch_raises(ctx):
    a = G.csr_fixed(10, 10, 2, 1)
    b = G.csr_fixed(10, 11, 2, 2)
    with pytest.raises(StamError) as e:
        ctx.spadd(_dev([a, b]))
    assert e.value.code == "DimensionMismatch"


def test_spadd_arity(ctx):
    a = G.csr_fixed(10, 10, 2, 1)
    with pytest.raises(StamError) as e:
        ctx.spadd(_dev([a]))
    assert e.value.code == "ArityMismatch"


def test_spadd_mid_rows_take_the_cta_path(ctx):
    # rows between a warp's staging (384) and the CTA path's 3072 entries, some
    # with many shared columns, plus rows on either side of both limits
    rng = np.random.default_rng(17)
    ops = []
    for k in range(4):
        lens = rng.integers(100, 900, size=300)
        lens[[0, 1, 2, 3]] = [96, 97, 800, 1000]
        pos = np.zeros(301, dtype=np.int64)
        np.cumsum(lens, out=pos[1:])
        ops.append(G.csr_from_lengths(300, 3000, pos, 500 + k))
    D = ctx.spadd(_dev(ops))
    oracle.compare_csr(D, oracle.spadd(ops), exact_values=True)
    # assemble mode through the same path
    Dz = ctx.spadd(_dev(ops), mode="assemble")
    assert np.array_equal(Dz.idx.cpu().numpy(), D.idx.cpu().numpy())


@pytest.mark.parametrize("k", [17, 33])
def test_spadd_more_operands_than_one_kernel_call(ctx, k):
    # > 16 operands: the workspace sequence continues across kernel calls with
    # the partial sum as operand 0 — bit-identical to one pass in order
    rng = np.random.default_rng(k)
    ops = []
    for q in range(k):
        lens = rng.integers(0, 12, size=300)
        pos = np.zeros(301, dtype=np.int64)
        np.cumsum(lens, out=pos[1:])
        ops.append(G.csr_from_lengths(300, 400, pos, 500 + q))
    D = ctx.spadd(_dev(ops), result="host")
    oracle.compare_csr(D, oracle.spadd(ops), exact_values=True)
