"""GPU parity under a dirty memory pool: small randomized SpGEMM and sparse
MTTKRP problems interleaved on one context, so every call's temporaries reuse
the previous calls' memory (a control word that a kernel reads before its
zeroing is ordered shows up here, not in a fresh process)."""
import numpy as np
import pytest

import oracle
from paper_1802_10574_b200 import generators as G

pytestmark = pytest.mark.gpu


def _d(x):
    return x.to("cuda")


def test_interleaved_calls_reuse_pool_memory(ctx):
    rng = np.random.default_rng(2024)
    big = G.make_config(3, scale=0.01)
    for it in range(6):
        # a larger call first: leaves non-zero temporaries behind
        ctx.spgemm(_d(big["A"]), _d(big["B"]))
        m = int(rng.integers(50, 400))
        n = int(rng.integers(2_000, 300_000))
        per_a = int(rng.integers(2, 60))
        per_b = int(rng.integers(1, 40))
        A = G.csr_fixed(m, 300, per_a, 100 + it)
        B = G.csr_fixed(300, n, per_b, 200 + it)
        C = ctx.spgemm(_d(A), _d(B))
        oracle.compare_csr(C, oracle.spgemm(A, B))
        # sparse MTTKRP on mostly single-nonzero fibers (the three-phase path)
        I = int(rng.integers(20, 200))
        sizes = rng.integers(0, 120, I).astype(np.int64)
        T = G.csf3((I, 5000, 700), sizes, 300 + it)
        R = int(rng.choice([32, 64, 128, 256]))
        per = int(rng.integers(2, max(3, R // 6)))
        Cf = G.csr_fixed(5000, R, per, 400 + it)
        Df = G.csr_fixed(700, R, per, 500 + it)
        Asp = ctx.mttkrp(_d(T), _d(Cf), _d(Df))
        oracle.compare_csr(Asp, oracle.mttkrp_sparse(T, Cf, Df))
