"""GPU: SpGEMM execution modes and unsorted output
 vs the CPU oracle.

* ASSEMBLE gives the exact index (pos/idx bit-identical to the oracle's) with
  zero values.
* COMPUTE into an assembled index is SPEC's compute-after-assemble: pos/idx
  unchanged, values bit-identical to the CPU workspace (canonical order), also
  for rows the fused path accumulates with atomics.
* sort=False keeps every row's column set (any order) and the values.
* A product whose column is missing from the index raises MissingSlot.
"""
import numpy as np
import pytest

import oracle
from paper_1802_10574_b200 import CSR, StamError
from paper_1802_10574_b200 import generators as G

pytestmark = pytest.mark.gpu


def _d(m):
    return m.to("cuda")


def _np(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def _rows_sorted(M):
    """Host copy of M with every row sorted by column (values carried)."""
    pos, idx, vals = _np(M.pos), _np(M.idx).copy(), _np(M.vals).copy()
    for i in range(M.nrows):
        b, e = pos[i], pos[i + 1]
        o = np.argsort(idx[b:e], kind="stable")
        idx[b:e] = idx[b:e][o]
        vals[b:e] = vals[b:e][o]
    return CSR(M.nrows, M.ncols, pos.copy(), idx, vals)


@pytest.fixture(scope="module")
def powerlaw():
    cfg = G.make_config(3, scale=0.01)  # every bin incl. long rows
    return cfg["A"], cfg["B"], oracle.spgemm(cfg["A"], cfg["B"], nthreads=oracle.threads_default())


def test_assemble_gives_exact_index_zero_values(ctx, powerlaw):
    A, B, ref = powerlaw
    C = ctx.spgemm(_d(A), _d(B), mode="assemble")
    assert np.array_equal(_np(C.pos), ref["pos"]) and np.array_equal(_np(C.idx), ref["idx"])
    assert not np.any(_np(C.vals))


def test_compute_after_assemble_is_bit_identical(ctx, powerlaw):
    A, B, ref = powerlaw
    idx = ctx.spgemm(_d(A), _d(B), mode="assemble")
    C = ctx.spgemm_compute(_d(A), _d(B), idx)
    rep = oracle.compare_csr(C, ref, exact_values=True)
    assert rep["bit_identical"]


def test_compute_reuses_one_index_for_new_values(ctx):
    # assemble once, compute many: same pattern, new values
    cfg = G.make_config(1, scale=0.05)
    A, B = cfg["A"], cfg["B"]
    idx = ctx.spgemm(_d(A), _d(B), mode="assemble", result="host")
    A2 = CSR(A.nrows, A.ncols, A.pos, A.idx, np.asarray(A.vals) * -0.5 + 0.25)
    C = ctx.spgemm_compute(A2, B, idx, result="host")
    oracle.compare_csr(C, oracle.spgemm(A2, B), exact_values=True)


def test_unsorted_fused_keeps_row_sets(ctx, powerlaw):
    A, B, ref = powerlaw
    C = ctx.spgemm(_d(A), _d(B), sort=False)
    assert np.array_equal(_np(C.pos), ref["pos"])
    oracle.compare_csr(_rows_sorted(C), ref)


def test_compute_into_unsorted_index(ctx, powerlaw):
    A, B, ref = powerlaw
    idx = ctx.spgemm(_d(A), _d(B), mode="assemble", sort=False)
    C = ctx.spgemm_compute(_d(A), _d(B), idx, sort=False)
    assert np.array_equal(_np(C.idx), _np(idx.idx))  # index untouched
    oracle.compare_csr(_rows_sorted(C), ref, exact_values=True)


def test_compute_missing_slot(ctx):
    cfg = G.make_config(1, scale=0.01)
    A, B = cfg["A"], cfg["B"]
    full = ctx.spgemm(A, B, mode="assemble", result="host")
    # drop the last entry of row 0
    pos, idx = _np(full.pos).copy(), _np(full.idx)
    keep = np.ones(idx.shape[0], dtype=bool)
    keep[pos[1] - 1] = False
    pos[1:] -= 1
    bad = CSR(full.nrows, full.ncols, pos, idx[keep].copy(), np.zeros(int(keep.sum())))
    with pytest.raises(StamError) as e:
        ctx.spgemm_compute(A, B, bad)
    assert e.value.code == "MissingSlot"


def test_compute_mode_flag_on_fused_entry_is_rejected(ctx):
    cfg = G.make_config(1, scale=0.01)
    with pytest.raises(StamError) as e:
        ctx.spgemm(cfg["A"], cfg["B"], mode="compute")
    assert e.value.code == "PreconditionViolated"


# --------------------------------------------------------------------------
# SpAdd: assemble / compute (operand order: operand 0 assigns, others
# accumulate; an entry first reached by a later operand accumulates into 0.0)

@pytest.fixture(scope="module")
def spadd_ops():
    rng = np.random.default_rng(5)
    ops = []
    for k in range(3):
        lens = rng.integers(0, 60, size=700)
        lens[[5, 99]] = [3000, 700]  # a deferred (long) row and a postponed one
        pos = np.zeros(701, dtype=np.int64)
        np.cumsum(lens, out=pos[1:])
        ops.append(G.csr_from_lengths(700, 4000, pos, 300 + k))  # narrow: many shared columns
    return ops, oracle.spadd(ops)


def test_spadd_assemble_exact_index(ctx, spadd_ops):
    ops, ref = spadd_ops
    D = ctx.spadd([_d(o) for o in ops], mode="assemble")
    assert np.array_equal(_np(D.pos), ref["pos"]) and np.array_equal(_np(D.idx), ref["idx"])
    assert not np.any(_np(D.vals))


def test_spadd_compute_after_assemble_bit_identical(ctx, spadd_ops):
    ops, ref = spadd_ops
    idx = ctx.spadd([_d(o) for o in ops], mode="assemble")
    D = ctx.spadd_compute([_d(o) for o in ops], idx)
    assert oracle.compare_csr(D, ref, exact_values=True)["bit_identical"]


def test_spadd_compute_unsorted_index_and_missing_slot(ctx, spadd_ops):
    ops, ref = spadd_ops
    idx = ctx.spadd(ops, mode="assemble", result="host")
    pos, cols = _np(idx.pos), _np(idx.idx).copy()
    for i in range(idx.nrows):  # reverse every row: a valid unsorted index
        cols[pos[i]:pos[i + 1]] = cols[pos[i]:pos[i + 1]][::-1]
    rev = CSR(idx.nrows, idx.ncols, pos.copy(), cols, np.zeros(cols.shape[0]))
    D = ctx.spadd_compute(ops, rev, sort=False, result="host")
    oracle.compare_csr(_rows_sorted(D), ref, exact_values=True)
    short = CSR(idx.nrows, idx.ncols, np.concatenate([[0], pos[1:] - 1]) if pos[1] > 0 else pos,
                np.delete(_np(idx.idx), 0) if pos[1] > 0 else _np(idx.idx),
                np.zeros(cols.shape[0] - (1 if pos[1] > 0 else 0)))
    if pos[1] > 0:
        with pytest.raises(StamError) as e:
            ctx.spadd_compute(ops, short)
        assert e.value.code == "MissingSlot"


# --------------------------------------------------------------------------
# exchange formats feeding the kernels

def test_loaded_files_through_the_kernels(ctx, tmp_path):
    from paper_1802_10574_b200 import io as sio

    A = G.csr_powerlaw(2000, 2000, 77, lmax=300)
    sio.store(tmp_path / "a.mtx", A)
    L = sio.load_matrix_market(tmp_path / "a.mtx")
    oracle.compare_csr(ctx.spgemm(_d(L), _d(L)), oracle.spgemm(A, A))
    B = G.csf3((50, 60, 70), G.slice_sizes_ranksize(50, 4000, 1.5, 3), 4)
    sio.store(tmp_path / "b.tns", B)
    T = sio.load_tns(tmp_path / "b.tns", dims=B.dims)
    Cf, Df = G.dense(60, 32, 5), G.dense(70, 32, 6)
    got = _np(ctx.mttkrp(T, Cf, Df).vals)
    ref = oracle.mttkrp_dense(B, Cf.vals, Df.vals)
    bound = 1e-12 * np.maximum(np.abs(ref["vals"]), ref["abs"])
    assert np.all(np.abs(got - ref["vals"]) <= bound)
