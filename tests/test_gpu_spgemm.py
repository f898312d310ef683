"""GPU parity: SpGEMM through the C ABI vs the CPU oracle.

Structure (pos, idx) must be bit-identical; values within the scaled
tolerance |x - x_ref| <= 1e-12 * max(|x_ref|, sum|terms|).  Rows
with at most 32 products accumulate in canonical order on the GPU and are
bit-identical too."""
import numpy as np
import pytest

import oracle
from paper_1802_10574_b200 import CSR, StamError
from paper_1802_10574_b200 import generators as G

pytestmark = pytest.mark.gpu


def _d(m):
    return m.to("cuda")


@pytest.mark.parametrize("scale", [0.01, 0.1])
def test_spgemm_config1_scaled(ctx, scale):
    cfg = G.make_config(1, scale=scale)
    C = ctx.spgemm(_d(cfg["A"]), _d(cfg["B"]))
    oracle.compare_csr(C, oracle.spgemm(cfg["A"], cfg["B"]))


def test_spgemm_config1_full(ctx):
    cfg = G.make_config(1)
    C = ctx.spgemm(_d(cfg["A"]), _d(cfg["B"]))
    oracle.compare_csr(C, oracle.spgemm(cfg["A"], cfg["B"], nthreads=oracle.threads_default()))


@pytest.mark.parametrize("scale", [0.002, 0.02])
def test_spgemm_config3_scaled(ctx, scale):
    # power-law rows: exercises every bin (tiny, hash S/M/L, long)
    cfg = G.make_config(3, scale=scale)
    C = ctx.spgemm(_d(cfg["A"]), _d(cfg["B"]))
    oracle.compare_csr(C, oracle.spgemm(cfg["A"], cfg["B"], nthreads=oracle.threads_default()))


def test_spgemm_identity(ctx):
    # identity x identity -> identity
    n = 1000
    I = CSR(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.ones(n))
    C = ctx.spgemm(_d(I), _d(I), result="host")
    assert np.array_equal(C.pos, I.pos) and np.array_equal(C.idx, I.idx)
    assert np.array_equal(C.vals, I.vals)


def test_spgemm_random_dense_oracle(ctx):
    # random 40x40 pair at density 0.1 equals the dense product
    rng = np.random.default_rng(40)
    a = rng.random((40, 40)) * (rng.random((40, 40)) < 0.1)
    b = rng.random((40, 40)) * (rng.random((40, 40)) < 0.1)
    C = ctx.spgemm(_d(CSR.from_dense(a)), _d(CSR.from_dense(b)), result="host")
    np.testing.assert_allclose(C.to_dense(), a @ b, rtol=1e-12, atol=1e-14)


def test_spgemm_rectangular_and_empty_rows(ctx):
    rng = np.random.default_rng(3)
    lens = rng.integers(0, 6, size=300)
    lens[rng.random(300) < 0.4] = 0
    pos = np.zeros(301, dtype=np.int64)
    np.cumsum(lens, out=pos[1:])
    A = G.csr_from_lengths(300, 200, pos, 5)
    lensb = rng.integers(0, 60, size=200)
    posb = np.zeros(201, dtype=np.int64)
    np.cumsum(lensb, out=posb[1:])
    B = G.csr_from_lengths(200, 5000, posb, 6)
    C = ctx.spgemm(_d(A), _d(B))
    oracle.compare_csr(C, oracle.spgemm(A, B))


def test_spgemm_every_bin_boundary(ctx):
    # rows with exactly the tier-boundary product counts (and one past each)
    targets = [0, 1, 32, 33, 64, 65, 256, 257, 1024, 1025, 2048, 2049, 4096, 4097, 8192, 8193, 20000]
    n = 200_000
    B = G.csr_fixed(n // 4, n, 1, 11)  # every B row has one entry
    pos = np.zeros(len(targets) + 1, dtype=np.int64)
    np.cumsum(targets, out=pos[1:])
    A = G.csr_from_lengths(len(targets), n // 4, pos, 12)
    C = ctx.spgemm(_d(A), _d(B))
    oracle.compare_csr(C, oracle.spgemm(A, B))


def test_spgemm_heavy_collisions(ctx):
    # narrow B column range: many products per output column
    A = G.csr_fixed(500, 400, 60, 21)
    B = G.csr_fixed(400, 64, 30, 22)
    C = ctx.spgemm(_d(A), _d(B))
    oracle.compare_csr(C, oracle.spgemm(A, B))


def test_spgemm_clustered_columns_and_duplicates(ctx):
    # the numeric pass sorts a row's products by order-preserving buckets of its
    # column span: rows whose columns cluster (one far outlier stretches the
    # span, so everything else shares a bucket) must fall back to the hash
    # kernel, and duplicates inside ordinary buckets must fold into one entry
    n = 1_000_000
    rows_b, cols_b = [], []
    for k in range(10):  # B rows 0..9: 30 consecutive columns each
        rows_b += [k] * 30
        cols_b += list(range(k * 30, k * 30 + 30))
    rows_b += [10]
    cols_b += [n - 1]  # B row 10: the outlier
    rows_b += [11] * 30
    cols_b += list(range(0, 30))  # B row 11 repeats row 0's columns
    for k in range(12, 40):  # B rows 12..39: 40 consecutive columns each, 20 apart (overlapping)
        rows_b += [k] * 40
        cols_b += list(range(5000 + (k - 12) * 20, 5000 + (k - 12) * 20 + 40))
    rng = np.random.default_rng(7)
    pos_b = np.zeros(41, dtype=np.int64)
    np.add.at(pos_b, np.asarray(rows_b) + 1, 1)
    pos_b = np.cumsum(pos_b)
    B = CSR(40, n, pos_b, np.asarray(cols_b, dtype=np.int64), rng.uniform(-1, 1, len(cols_b)))
    a_rows = [list(range(11)),        # 301 products, 300 of them in one bucket -> hash kernel
              [0, 10, 11],            # 61 products, 30 duplicated, clustered
              [0, 11],                # 60 products over 30 columns: duplicates in every bucket
              list(range(12, 40)),    # 1120 products, every column held twice (overlapping rows)
              list(range(0, 40))]     # 1481 products, everything at once
    pos_a = np.zeros(len(a_rows) + 1, dtype=np.int64)
    pos_a[1:] = np.cumsum([len(r) for r in a_rows])
    idx_a = np.concatenate([np.asarray(r, dtype=np.int64) for r in a_rows])
    A = CSR(len(a_rows), 40, pos_a, idx_a, rng.uniform(-1, 1, len(idx_a)))
    C = ctx.spgemm(_d(A), _d(B))
    oracle.compare_csr(C, oracle.spgemm(A, B))


def test_spgemm_tiny_rows_bit_exact(ctx):
    A = G.csr_fixed(2000, 3000, 3, 31)
    B = G.csr_fixed(3000, 50, 8, 32)  # <= 24 products per row, many collisions
    C = ctx.spgemm(_d(A), _d(B))
    rep = oracle.compare_csr(C, oracle.spgemm(A, B), exact_values=True)
    assert rep["bit_identical"]


def test_spgemm_host_io(ctx):
    cfg = G.make_config(1, scale=0.05)
    C = ctx.spgemm(cfg["A"], cfg["B"], result="host")
    assert isinstance(C.idx, np.ndarray)
    oracle.compare_csr(C, oracle.spgemm(cfg["A"], cfg["B"]))


def test_spgemm_dimension_mismatch(ctx):
    A = G.csr_fixed(10, 12, 2, 1)
    B = G.csr_fixed(10, 10, 2, 2)
    with pytest.raises(StamError) as e:
        ctx.spgemm(_d(A), _d(B))
    assert e.value.code == "DimensionMismatch"


def test_spgemm_counters(ctx):
    # Gustavson mults = sum over stored A(i,k) of nnz(B_k)
    from paper_1802_10574_b200 import _native as N

    cfg = G.make_config(1, scale=0.05)
    st = N.Stats()
    ctx.spgemm(_d(cfg["A"]), _d(cfg["B"]), stats=st)
    A, B = cfg["A"], cfg["B"]
    expect = int(np.sum(np.diff(B.pos)[A.idx]))
    assert st.mults == expect
    assert st.appends == ctx.spgemm(_d(A), _d(B)).nnz


def test_spgemm_wide_long_rows_column_windows(ctx):
    # B has 3M columns (wider than a shared-memory bitmap): rows with more than
    # 4096 products take the long-row path in column windows
    rng = np.random.default_rng(21)
    n, used, per_b, m, per_a = 3_000_000, 1000, 100, 48, 80
    blens = np.zeros(n, dtype=np.int64)
    blens[:used] = per_b
    bpos = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(blens, out=bpos[1:])
    B = G.csr_from_lengths(n, n, bpos, 22)
    aidx = np.concatenate([np.sort(rng.choice(used, per_a, replace=False)) for _ in range(m)])
    A = CSR(m, n, np.arange(m + 1, dtype=np.int64) * per_a, aidx.astype(np.int64),
            rng.uniform(-1, 1, m * per_a))
    C = ctx.spgemm(_d(A), _d(B))
    oracle.compare_csr(C, oracle.spgemm(A, B, nthreads=oracle.threads_default()))
