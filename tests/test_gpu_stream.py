"""Host-streamed calls (host inputs / host result above the streaming
thresholds): SpGEMM row blocks downloaded while later blocks compute, sparse
MTTKRP slice blocks uploaded and downloaded around the device path.  Each must
equal the oracle like the device path does (structure bit-exact, values within
the scaled 1e-12 bound)."""
import os

import numpy as np
import pytest

import oracle
from paper_1802_10574_b200 import _native as N
from paper_1802_10574_b200 import generators as G

pytestmark = pytest.mark.gpu

NT = os.cpu_count() or 1


def test_spgemm_host_result_streams_row_blocks(ctx):
    A = G.make_config(3, scale=0.3)["A"]  # 300k rows, ~4.9M nnz: above the streaming threshold
    assert A.nrows >= 65536 and A.nnz >= 1 << 22
    st = N.Stats()
    C = ctx.spgemm(A, A, result="host", stats=st)
    ref = oracle.spgemm(A, A, nthreads=NT)
    oracle.compare_csr(C, ref)
    assert st.kernel_launches > 16  # eight blocks, each a device pipeline


def test_mttkrp_sparse_host_inputs_stream_slice_blocks(ctx):
    cfg = G.make_config(5, scale=0.1)  # 50k slices, 20M nonzeros
    B = cfg["B"]
    assert B.nnz >= 1 << 24
    st = N.Stats()
    A = ctx.mttkrp(B, cfg["C"], cfg["D"], result="host", stats=st)
    ref = oracle.mttkrp_sparse(B, cfg["C"], cfg["D"], nthreads=NT)
    oracle.compare_csr(A, ref)
    # the SPEC counter is the sum over blocks
    dev = ctx.mttkrp(B.to("cuda"), cfg["C"].to("cuda"), cfg["D"].to("cuda"))
    assert dev.nnz == A.nnz


def test_mttkrp_sparse_bounded_staging_blocks(ctx, monkeypatch):
    """A staging budget below 16·I·R bytes splits the slices into blocks whose
    results are placed into one exact CSR (ADVICE: bounded staging memory)."""
    cfg = G.make_config(5, scale=0.01)  # 5k slices, R = 256: 20 MB of staging unblocked
    monkeypatch.setenv("STAM_SPARSE_STAGE_MB", "2")  # -> 512 slices per block
    st = N.Stats()
    A = ctx.mttkrp(cfg["B"].to("cuda"), cfg["C"].to("cuda"), cfg["D"].to("cuda"), stats=st)
    ref = oracle.mttkrp_sparse(cfg["B"], cfg["C"], cfg["D"], nthreads=NT)
    oracle.compare_csr(A, ref)
    monkeypatch.delenv("STAM_SPARSE_STAGE_MB")
    st1 = N.Stats()
    A1 = ctx.mttkrp(cfg["B"].to("cuda"), cfg["C"].to("cuda"), cfg["D"].to("cuda"), stats=st1)
    assert A1.nnz == A.nnz and st.mults == st1.mults
    assert st.kernel_launches > st1.kernel_launches  # ten blocks, each a device call
