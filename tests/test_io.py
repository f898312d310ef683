"""Exchange formats: Python loaders vs the SPEC examples,
round trips, and agreement with the C++ loaders (tests/cpp/test_api.cpp)."""
import numpy as np
import pytest

from paper_1802_10574_b200 import CSR, StamError
from paper_1802_10574_b200 import generators as G
from paper_1802_10574_b200 import io as sio


def _w(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return p


def test_mtx_identity_and_symmetric_expansion(tmp_path):
    I = sio.load_matrix_market(_w(tmp_path, "i.mtx",
                                  "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 2 1\n"))
    assert I.pos.tolist() == [0, 1, 2] and I.idx.tolist() == [0, 1] and I.vals.tolist() == [1, 1]
    S = sio.load_matrix_market(_w(tmp_path, "s.mtx",
                                  "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 5\n3 3 1\n"))
    assert S.nnz == 3 and S.pos.tolist() == [0, 1, 2, 3] and S.idx.tolist() == [1, 0, 2]
    K = sio.load_matrix_market(_w(tmp_path, "k.mtx",
                                  "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 3\n"))
    assert K.vals.tolist() == [-3.0, 3.0]


def test_mtx_errors(tmp_path):
    with pytest.raises(StamError) as e:
        sio.load_matrix_market(_w(tmp_path, "b.mtx", "%%MatrixMarket tensor coordinate real general\n"))
    assert e.value.code == "Io" and ":1:" in str(e.value)
    with pytest.raises(StamError) as e:
        sio.load_matrix_market(_w(tmp_path, "o.mtx",
                                  "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n"))
    assert e.value.code == "OutOfRange"


def test_tns_duplicates_and_zero_based(tmp_path):
    T = sio.load_tns(_w(tmp_path, "t.tns", "# c\n1 1 1 1.5\n2 3 1 2\n1 1 1 0.5\n1 2 2 3\n"))
    assert T.nnz == 3 and T.dims == (2, 3, 2) and T.vals[0] == 2.0
    with pytest.raises(StamError) as e:
        sio.load_tns(_w(tmp_path, "z.tns", "0 1 1 1\n"))
    assert e.value.code == "OutOfRange"


@pytest.mark.parametrize("seed", range(5))
def test_round_trips(tmp_path, seed):
    A = G.csr_powerlaw(300, 200, seed, lmax=50)
    sio.store(tmp_path / "a.mtx", A)
    B = sio.load_matrix_market(tmp_path / "a.mtx")
    assert np.array_equal(B.pos, A.pos) and np.array_equal(B.idx, A.idx)
    assert np.array_equal(B.vals.view(np.int64), np.asarray(A.vals).view(np.int64))
    T = G.csf3((20, 30, 40), G.slice_sizes_ranksize(20, 500, 1.5, seed), seed)
    sio.store(tmp_path / "t.tns", T)
    U = sio.load_tns(tmp_path / "t.tns", dims=T.dims)
    for f in ("pos1", "idx1", "pos2", "idx2"):
        assert np.array_equal(getattr(U, f), getattr(T, f)), f
    assert np.array_equal(U.vals.view(np.int64), np.asarray(T.vals).view(np.int64))
