"""GPU: CIN-driven dispatch end to end — the golden printed statements run
through paper_1802_10574_b200.execute and match the CPU oracle."""
import numpy as np
import pytest

import oracle
from paper_1802_10574_b200 import generators as G
from paper_1802_10574_b200.execute import execute

pytestmark = pytest.mark.gpu

SPGEMM = "forall(i) ((forall(j) A(i,j) = w0(j)) where (forall(k,j) w0(j) += B(i,k)*C(k,j)))"
SPADD = ("forall(i) ((forall(j) A(i,j) = w0(j)) where ((forall(j) w0(j) = B(i,j) ; forall(j) "
         "w0(j) += C(i,j) ; forall(j) w0(j) += D(i,j))))")
MTTKRP_S = ("forall(i) ((forall(j) A(i,j) = w1(j)) where (forall(k) ((forall(j) w1(j) += "
            "w0(j)*D(k,j)) where (forall(l,j) w0(j) += B(i,k,l)*C(l,j)))))")


def test_execute_spgemm_and_spadd(ctx):
    cfg = G.make_config(3, scale=0.005)
    name, plan, C = execute(SPGEMM, {"B": cfg["A"], "C": cfg["A"]}, ctx)
    assert (name, plan) == ("A", "spgemm")
    oracle.compare_csr(C, oracle.spgemm(cfg["A"], cfg["A"]))
    ops = G.make_config(2, scale=0.01)["ops"]
    name, plan, D = execute(SPADD, dict(zip("BCD", ops)), ctx)
    assert plan == "spadd"
    oracle.compare_csr(D, oracle.spadd(ops), exact_values=True)


def test_execute_mttkrp_sparse_golden_naming(ctx):
    cfg = G.make_config(5, scale=0.002)
    B, Cf, Df = cfg["B"], cfg["C"], cfg["D"]  # API: C middle mode, D innermost
    # golden naming: D(k,j) is the middle-mode factor, C(l,j) the innermost
    name, plan, A = execute(MTTKRP_S, {"B": B, "D": Cf, "C": Df}, ctx)
    assert plan == "mttkrp_sparse"
    oracle.compare_csr(A, oracle.mttkrp_sparse(B, Cf, Df))
