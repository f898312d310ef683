"""CPU: CIN parsing and plan matching (paper_1802_10574_b200.execute) on the
golden printed statements of the reference's schedule() tests
(tests/test_transform.cpp:141-147, 166-184, 275-284), renamed variables, and
the SPEC rejections (3-way merge without a workspace, scattered sparse
inserts, parse errors)."""
import pytest

from paper_1802_10574_b200 import StamError
from paper_1802_10574_b200.execute import match, parse

GOLDEN = {
    "spgemm": "forall(i) ((forall(j) A(i,j) = w0(j)) where (forall(k,j) w0(j) += B(i,k)*C(k,j)))",
    "mttkrp_dense": "forall(i,k) ((forall(j) A(i,j) += w0(j)*D(k,j)) where (forall(l,j) w0(j) += "
                    "B(i,k,l)*C(l,j)))",
    "mttkrp_sparse": "forall(i) ((forall(j) A(i,j) = w1(j)) where (forall(k) ((forall(j) w1(j) += "
                     "w0(j)*D(k,j)) where (forall(l,j) w0(j) += B(i,k,l)*C(l,j)))))",
    "spadd": "forall(i) ((forall(j) A(i,j) = w0(j)) where ((forall(j) w0(j) = B(i,j) ; forall(j) "
             "w0(j) += C(i,j) ; forall(j) w0(j) += D(i,j))))",
    "ttv": "forall(i,j,k) A(i,j) += B(i,j,k)*c(k)",
    "rowdot": "forall(i,j) a(i) += B(i,j)*C(i,j)",
    "spadd_merge": "forall(i,j) A(i,j) = B(i,j) + C(i,j)",
}


@pytest.mark.parametrize("plan", sorted(GOLDEN))
def test_golden_statements_match(plan):
    pl = match(parse(GOLDEN[plan]))
    assert pl.plan == plan
    assert pl.tensor in ("A", "a")


def test_mttkrp_factor_roles():
    pl = match(parse(GOLDEN["mttkrp_dense"]))
    assert pl.args == ("B", "D", "C")  # the middle mode's factor first (API order)


def test_renamed_variables_and_tensors():
    pl = match(parse("forall(r) ((forall(c) Out(r,c) = acc(c)) where "
                     "(forall(m,c) acc(c) += X(r,m)*Y(m,c)))"))
    assert (pl.plan, pl.tensor, pl.args) == ("spgemm", "Out", ("X", "Y"))


def test_rejections():
    with pytest.raises(StamError) as e:
        match(parse("forall(i,j) A(i,j) = B(i,j) + C(i,j) + D(i,j)"))
    assert e.value.code == "UnsupportedMerge"
    with pytest.raises(StamError) as e:
        match(parse("forall(i,k,j) A(i,j) += B(i,k)*C(k,j)"))
    assert e.value.code == "UnplannableResult"
    with pytest.raises(StamError) as e:
        parse("forall(i) (A(i) = ")
    assert e.value.code == "Parse"
    with pytest.raises(StamError) as e:  # wrong index pattern: no plan
        match(parse("forall(i) ((forall(j) A(i,j) = w0(j)) where (forall(k,j) w0(j) += "
                    "B(k,i)*C(k,j)))"))
    assert e.value.code == "UnsupportedMerge"
