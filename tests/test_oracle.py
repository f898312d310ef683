"""CPU: the oracle restatement (oracle/stam_oracle.c) pinned to the reference.

* bit-identical to the golden outputs of the reference's own Workspace /
  TensorBuilder (tests/golden, made by tests/golden/make_golden.py);
* bit-identical to oracle/_ref on fresh seeded inputs (when built here);
* equal to a dense evaluation (SPEC.md:450-470 dense oracle) on tiny inputs;
* SPEC counter formulas and thread-count invariance."""
import numpy as np
import pytest

import oracle
from _golden import load, names
from paper_1802_10574_b200 import CSF3, CSR
from paper_1802_10574_b200 import generators as G


def _run_port(kind, args):
    if kind == "spgemm":
        return oracle.spgemm(*args)
    if kind == "spadd":
        return oracle.spadd(*args)
    if kind == "mttkrp_dense":
        return oracle.mttkrp_dense(args[0], args[1].vals, args[2].vals)
    return oracle.mttkrp_sparse(*args)


@pytest.mark.parametrize("name", names())
def test_oracle_matches_reference_golden(name):
    kind, args, ref = load(name)
    got = _run_port(kind, args)
    if kind == "mttkrp_dense":
        assert np.array_equal(got["vals"].view(np.int64), ref["vals"].view(np.int64))
    else:
        rep = oracle.compare_csr(got, ref, exact_values=True)
        assert rep["bit_identical"]


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cid,scale", [(1, 0.05), (2, 0.002), (3, 0.002)])
def test_oracle_matches_reference_fresh_inputs(cid, scale):
    cfg = G.make_config(cid, scale=scale)
    if cfg["kind"] == "spgemm":
        a, b = oracle.spgemm(cfg["A"], cfg["B"]), oracle.ref_spgemm(cfg["A"], cfg["B"], 3)
    else:
        a, b = oracle.spadd(cfg["ops"]), oracle.ref_spadd(cfg["ops"], 3)
    assert oracle.compare_csr(a, b, exact_values=True)["bit_identical"]


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_oracle_matches_reference_mttkrp_fresh():
    cfg = G.make_config(4, scale=0.01)
    a = oracle.mttkrp_dense(cfg["B"], cfg["C"].vals, cfg["D"].vals, 2)
    b = oracle.ref_mttkrp_dense(cfg["B"], cfg["C"].vals, cfg["D"].vals, 3)
    assert np.array_equal(a["vals"].view(np.int64), b["vals"].view(np.int64))
    cfg = G.make_config(5, scale=0.0005)
    a = oracle.mttkrp_sparse(cfg["B"], cfg["C"], cfg["D"], 2)
    b = oracle.ref_mttkrp_sparse(cfg["B"], cfg["C"], cfg["D"], 3)
    assert oracle.compare_csr(a, b, exact_values=True)["bit_identical"]


def test_dense_evaluation_spgemm_spadd():
    rng = np.random.default_rng(0)
    a = rng.random((30, 20)) * (rng.random((30, 20)) < 0.2)
    b = rng.random((20, 25)) * (rng.random((20, 25)) < 0.2)
    c = oracle.spgemm(CSR.from_dense(a), CSR.from_dense(b))
    got = CSR(30, 25, c["pos"], c["idx"], c["vals"]).to_dense()
    np.testing.assert_allclose(got, a @ b, rtol=1e-14, atol=1e-15)
    ms = [rng.random((10, 10)) * (rng.random((10, 10)) < 0.3) for _ in range(3)]
    d = oracle.spadd([CSR.from_dense(m) for m in ms])
    np.testing.assert_allclose(CSR(10, 10, d["pos"], d["idx"], d["vals"]).to_dense(), sum(ms))


def test_dense_evaluation_mttkrp():
    rng = np.random.default_rng(1)
    t = rng.random((4, 5, 6)) * (rng.random((4, 5, 6)) < 0.4)
    C, D = rng.random((5, 3)), rng.random((6, 3))
    got = oracle.mttkrp_dense(CSF3.from_dense(t), C, D)["vals"]
    np.testing.assert_allclose(got, np.einsum("ijk,jr,kr->ir", t, C, D), rtol=1e-13)


def test_spec_row_dot_known_answer():
    # a_i = sum_j B_ij C_ij with B = C = [[1,2],[3,4]] -> [5, 25],
    # as the diagonal of B*C^T through the SpGEMM workspace kernel
    B = CSR.from_dense(np.array([[1.0, 2.0], [3.0, 4.0]]))
    Ct = CSR.from_dense(np.array([[1.0, 3.0], [2.0, 4.0]]))
    out = oracle.spgemm(B, Ct)
    dense = CSR(2, 2, out["pos"], out["idx"], out["vals"]).to_dense()
    assert list(np.diag(dense)) == [5.0, 25.0]


def test_spec_counters():
    # Gustavson mults = sum_{(i,k) in A} nnz(B_k)
    cfg = G.make_config(1, scale=0.02)
    A, B = cfg["A"], cfg["B"]
    oracle.spgemm(A, B)
    assert oracle.last_counters()["mults"] == int(np.sum(np.diff(B.pos)[A.idx]))
    # MTTKRP: hoisted mults = nnz*R + fibers*R (vs 2*nnz*R before the workspace)
    cfg = G.make_config(4, scale=0.005)
    oracle.mttkrp_dense(cfg["B"], cfg["C"].vals, cfg["D"].vals)
    R = cfg["C"].ncols
    assert oracle.last_counters()["mults"] == (cfg["B"].nnz + cfg["B"].nfibers) * R


@pytest.mark.parametrize("nt", [1, 3, 8])
def test_oracle_thread_invariance(nt):
    cfg = G.make_config(3, scale=0.001)
    base = oracle.spgemm(cfg["A"], cfg["B"], 1)
    assert oracle.compare_csr(oracle.spgemm(cfg["A"], cfg["B"], nt), base,
                              exact_values=True)["bit_identical"]


def test_spadd_signed_zero_rules():
    # workspace: op0 assigns (keeps -0.0), later operands accumulate into 0.0
    a = CSR(1, 3, np.array([0, 1]), np.array([0]), np.array([-0.0]))
    b = CSR(1, 3, np.array([0, 1]), np.array([1]), np.array([-0.0]))
    for m in (a, b):
        m.pos, m.idx = m.pos.astype(np.int64), m.idx.astype(np.int64)
    out = oracle.spadd([a, b])
    assert np.signbit(out["vals"][0]) and not np.signbit(out["vals"][1])
