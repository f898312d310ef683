"""GPU vs the reference's own outputs (tests/golden, generated through the
reference's stam::Workspace / TensorBuilder).  Structure bit-exact; values
bit-exact where the kernel accumulates in canonical order (SpAdd, tiny SpGEMM
rows), otherwise within the scaled 1e-12 tolerance."""
import numpy as np
import pytest

import oracle
from _golden import load, names

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", names())
def test_gpu_matches_reference_golden(ctx, name):
    kind, args, ref = load(name)
    dev = [a.to("cuda") if hasattr(a, "to") else [x.to("cuda") for x in a] for a in args]
    if kind == "spgemm":
        got = ctx.spgemm(*dev)
        ref["abs"] = oracle.spgemm(*args)["abs"]
        oracle.compare_csr(got, ref)
    elif kind == "spadd":
        got = ctx.spadd(dev[0])
        oracle.compare_csr(got, ref, exact_values=True)
    elif kind == "mttkrp_dense":
        got = ctx.mttkrp(*dev).numpy()
        port = oracle.mttkrp_dense(args[0], args[1].vals, args[2].vals)
        err = np.abs(got - ref["vals"])
        assert np.all(err <= 1e-12 * np.maximum(np.abs(ref["vals"]), port["abs"]))
    else:
        got = ctx.mttkrp(*dev)
        ref["abs"] = oracle.mttkrp_sparse(*args)["abs"]
        oracle.compare_csr(got, ref)
