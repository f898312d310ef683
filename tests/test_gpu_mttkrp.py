"""GPU parity: CSF MTTKRP (dense and sparse result) vs the CPU oracle.

Values within |x - x_ref| <= 1e-12 * max(|x_ref|, s_ref), s_ref the sum of
|terms| (reordering 6k-term sums breaks a per-entry 1e-12
relative bound, the scaled bound holds); sparse-result structure bit-exact
(presence-checked w0)."""
import numpy as np
import pytest

import oracle
from paper_1802_10574_b200 import CSF3, CSR, Dense, StamError
from paper_1802_10574_b200 import generators as G

pytestmark = pytest.mark.gpu


def _dense_ok(A, ref, tol=1e-12):
    got = A.numpy() if isinstance(A, Dense) else np.asarray(A)
    err = np.abs(got - ref["vals"])
    bound = tol * np.maximum(np.abs(ref["vals"]), ref["abs"])
    assert np.all(err <= bound), f"{int(np.sum(err > bound))} entries out of tolerance"


def _d(x):
    return x.to("cuda")


@pytest.mark.parametrize("scale", [0.005, 0.05])
def test_mttkrp_dense_config4_scaled(ctx, scale):
    cfg = G.make_config(4, scale=scale)
    A = ctx.mttkrp(_d(cfg["B"]), _d(cfg["C"]), _d(cfg["D"]))
    _dense_ok(A, oracle.mttkrp_dense(cfg["B"], cfg["C"].vals, cfg["D"].vals, 8))


@pytest.mark.slow
def test_mttkrp_dense_config4_full(ctx):
    cfg = G.make_config(4)
    A = ctx.mttkrp(_d(cfg["B"]), _d(cfg["C"]), _d(cfg["D"]))
    _dense_ok(A, oracle.mttkrp_dense(cfg["B"], cfg["C"].vals, cfg["D"].vals,
                                     oracle.threads_default()))


@pytest.mark.parametrize("R", [1, 7, 32, 33, 64, 100])
def test_mttkrp_dense_ranks(ctx, R):
    sizes = G.slice_sizes_ranksize(300, 20000, 1.5, 5)
    B = G.csf3((300, 200, 400), sizes, 6)
    C = G.dense(200, R, 7)
    D = G.dense(400, R, 8)
    A = ctx.mttkrp(_d(B), _d(C), _d(D))
    _dense_ok(A, oracle.mttkrp_dense(B, C.vals, D.vals))


def test_mttkrp_dense_empty_slices_and_long_fibers(ctx):
    # one slice with very long fibers (crosses many chunks), empty slices
    sizes = np.zeros(50, dtype=np.int64)
    sizes[[3, 10, 11, 40]] = [200_000, 5, 1, 3000]
    B = G.csf3((50, 20, 100_000), sizes, 9)
    C, D = G.dense(20, 32, 10), G.dense(100_000, 32, 11)
    A = ctx.mttkrp(_d(B), _d(C), _d(D))
    ref = oracle.mttkrp_dense(B, C.vals, D.vals)
    _dense_ok(A, ref)
    assert np.all(ref["vals"][[0, 1, 2, 49]] == 0)


def test_mttkrp_dense_matches_dense_einsum(ctx):
    rng = np.random.default_rng(1)
    t = rng.random((6, 5, 7)) * (rng.random((6, 5, 7)) < 0.3)
    C, D = rng.random((5, 4)), rng.random((7, 4))
    A = ctx.mttkrp(_d(CSF3.from_dense(t)), _d(Dense(C)), _d(Dense(D)), result="host")
    np.testing.assert_allclose(A.numpy(), np.einsum("ijk,jr,kr->ir", t, C, D), rtol=1e-12,
                               atol=1e-14)


def test_mttkrp_dense_deterministic(ctx):
    cfg = G.make_config(4, scale=0.02)
    args = (_d(cfg["B"]), _d(cfg["C"]), _d(cfg["D"]))
    a1 = ctx.mttkrp(*args).numpy()
    a2 = ctx.mttkrp(*args).numpy()
    assert np.array_equal(a1.view(np.int64), a2.view(np.int64))


@pytest.mark.parametrize("scale", [0.0005, 0.005])
def test_mttkrp_sparse_config5_scaled(ctx, scale):
    cfg = G.make_config(5, scale=scale)
    A = ctx.mttkrp(_d(cfg["B"]), _d(cfg["C"]), _d(cfg["D"]))
    oracle.compare_csr(A, oracle.mttkrp_sparse(cfg["B"], cfg["C"], cfg["D"], 8))


def test_mttkrp_sparse_multi_nonzero_fibers(ctx):
    # dense-ish slices: fibers with many k, factors with many columns per row
    sizes = np.full(40, 600, dtype=np.int64)
    B = G.csf3((40, 30, 50), sizes, 12)
    C = G.csr_fixed(30, 96, 40, 13)
    D = G.csr_fixed(50, 96, 25, 14)
    A = ctx.mttkrp(_d(B), _d(C), _d(D))
    oracle.compare_csr(A, oracle.mttkrp_sparse(B, C, D))


@pytest.mark.parametrize("per_row,sizes", [(6, 60), (24, 60), (3, 400), (40, 12)])
def test_mttkrp_sparse_three_phase_edges(ctx, per_row, sizes):
    # mostly single-nonzero fibers (the three-phase path) with some longer
    # fibers among them: sparse factors (few matches), dense factors (more hits
    # and matches than a slice's rows hold, columns shared by two nonzeros of
    # a fiber -> those slices take the single-pass kernel), long slices, and
    # the SPEC multiplication counter across all of them
    from paper_1802_10574_b200 import _native as N

    B = G.csf3((300, 6000, 450), np.full(300, sizes, dtype=np.int64), 21)
    assert B.nnz <= B.nfibers + B.nfibers // 8  # the three-phase path's condition
    C = G.csr_fixed(6000, 64, per_row, 22)
    D = G.csr_fixed(450, 64, per_row, 23)
    st = N.Stats()
    A = ctx.mttkrp(_d(B), _d(C), _d(D), stats=st)
    oracle.compare_csr(A, oracle.mttkrp_sparse(B, C, D))
    assert st.mults == oracle.last_counters()["mults"]


@pytest.mark.parametrize("R", [40, 320, 512])
def test_mttkrp_sparse_three_phase_ranks(ctx, R):
    # ranks off the 64-column word boundary and the widest bitmaps (8 words)
    from paper_1802_10574_b200 import _native as N

    B = G.csf3((400, 3000, 2500), np.full(400, 150, dtype=np.int64), 51)
    assert B.nnz <= B.nfibers + B.nfibers // 8
    C = G.csr_fixed(3000, R, max(3, R // 20), 52)
    D = G.csr_fixed(2500, R, max(3, R // 20), 53)
    st = N.Stats()
    A = ctx.mttkrp(_d(B), _d(C), _d(D), stats=st)
    oracle.compare_csr(A, oracle.mttkrp_sparse(B, C, D))
    assert st.mults == oracle.last_counters()["mults"]


def test_mttkrp_sparse_empty_slices_and_unaligned_views(ctx):
    # slices without fibers (leading, trailing, in runs) and CSF arrays that do
    # not start on a 16-byte boundary (bulk copies are replaced by lane copies)
    import torch

    sizes = np.zeros(257, dtype=np.int64)
    sizes[[3, 4, 40, 41, 42, 200]] = [70, 1, 33, 64, 5, 90]
    B = G.csf3((257, 300, 310), sizes, 31)
    C = G.csr_fixed(300, 128, 8, 32)
    D = G.csr_fixed(310, 128, 8, 33)
    want = oracle.mttkrp_sparse(B, C, D)
    oracle.compare_csr(ctx.mttkrp(_d(B), _d(C), _d(D)), want)

    def shifted(a):
        buf = torch.empty(len(a) + 1, dtype=torch.from_numpy(a).dtype, device="cuda")
        buf[1:].copy_(torch.from_numpy(a))
        return buf[1:]

    Bd = _d(B)
    Bu = type(Bd)(Bd.dims, Bd.pos1, shifted(B.idx1), shifted(B.pos2), shifted(B.idx2), shifted(B.vals))
    assert Bu.idx1.data_ptr() % 16 == 8
    oracle.compare_csr(ctx.mttkrp(Bu, _d(C), _d(D)), want)


def test_mttkrp_sparse_matches_dense_where_present(ctx):
    rng = np.random.default_rng(2)
    t = rng.random((5, 6, 7)) * (rng.random((5, 6, 7)) < 0.4)
    c = rng.random((6, 9)) * (rng.random((6, 9)) < 0.5)
    d = rng.random((7, 9)) * (rng.random((7, 9)) < 0.5)
    A = ctx.mttkrp(_d(CSF3.from_dense(t)), _d(CSR.from_dense(c)), _d(CSR.from_dense(d)),
                   result="host")
    np.testing.assert_allclose(A.to_dense(), np.einsum("ijk,jr,kr->ir", t, c, d), rtol=1e-12,
                               atol=1e-14)


def test_mttkrp_mixed_factors_rejected(ctx):
    cfg = G.make_config(4, scale=0.005)
    with pytest.raises(StamError):
        ctx.mttkrp(_d(cfg["B"]), _d(cfg["C"]), CSR.from_dense(np.eye(3)))


def test_mttkrp_dimension_mismatch(ctx):
    cfg = G.make_config(4, scale=0.005)
    with pytest.raises(StamError) as e:
        ctx.mttkrp(_d(cfg["B"]), _d(cfg["D"]), _d(cfg["C"]))
    assert e.value.code == "DimensionMismatch"


def test_mttkrp_sparse_counters_match_reference_formula(ctx):
    # SPEC.md:414-418 style counter: mults = sum over nonzeros of |D_k| (w0
    # inserts) + consumed w0 entries (presence-checked w1 updates)
    from paper_1802_10574_b200 import _native as N

    cfg = G.make_config(5, scale=0.0005)
    st = N.Stats()
    ctx.mttkrp(_d(cfg["B"]), _d(cfg["C"]), _d(cfg["D"]), stats=st)
    oracle.mttkrp_sparse(cfg["B"], cfg["C"], cfg["D"])
    assert st.mults == oracle.last_counters()["mults"]
