"""CPU: the Python storage mirror and the seeded generators."""
import numpy as np
import pytest

from paper_1802_10574_b200 import CSF3, CSR, StamError
from paper_1802_10574_b200 import generators as G


def test_csr_validate_catches_broken_invariants():
    good = CSR(2, 3, np.array([0, 1, 3]), np.array([2, 0, 1]), np.array([1.0, 2.0, 3.0]))
    good.validate()
    bad = CSR(2, 3, np.array([0, 2, 3]), np.array([2, 0, 1]), np.array([1.0, 2.0, 3.0]))
    with pytest.raises(StamError) as e:
        bad.validate()
    assert e.value.code == "Internal"


def test_dense_round_trips():
    rng = np.random.default_rng(3)
    m = rng.random((7, 9)) * (rng.random((7, 9)) < 0.4)
    assert np.array_equal(CSR.from_dense(m).to_dense(), m)
    t = rng.random((3, 4, 5)) * (rng.random((3, 4, 5)) < 0.3)
    b = CSF3.from_dense(t)
    b.validate()
    assert np.array_equal(b.to_dense(), t)


def test_view_requires_int64_and_f64():
    m = CSR(2, 2, np.array([0, 1, 2], dtype=np.int32), np.array([0, 1]), np.array([1.0, 2.0]))
    with pytest.raises(StamError):
        m.view()


def test_generators_are_deterministic_sorted_distinct():
    a = G.csr_fixed(100, 1000, 20, 5)
    b = G.csr_fixed(100, 1000, 20, 5)
    assert np.array_equal(a.idx, b.idx) and np.array_equal(a.vals, b.vals)
    a.validate()
    assert a.vals.min() >= -1 and a.vals.max() < 1
    c = G.csr_fixed(100, 1000, 20, 6)
    assert not np.array_equal(a.idx, c.idx)


def test_powerlaw_rows_match_the_stated_law():
    # config 3: P(L) ∝ (L + 1.7764)^-2 on [1, 5000], mean 16
    A = G.csr_powerlaw(200_000, 1_000_000, 301)
    lens = np.diff(A.pos)
    assert lens.min() >= 1 and lens.max() <= 5000
    assert 14.0 < lens.mean() < 18.0
    A.validate()


def test_ranksize_slices():
    s = G.slice_sizes_ranksize(12_092, 76_879_419, 1.5, 404)
    assert s.sum() == 76_879_419 and s.min() >= 1
    assert abs(s.max() / s.sum() - 0.385) < 0.01  # largest slice ~38.5%


def test_csf_generator_structure():
    sizes = G.slice_sizes_ranksize(50, 20_000, 1.5, 1)
    B = G.csf3((50, 100, 200), sizes, 2)
    B.validate()
    assert B.nnz == 20_000
    assert np.array_equal(np.diff(B.pos1) > 0, sizes > 0)
