"""Paper SpAdd experiment (PAPER.md:1705-1732 design): k
operands (k = 2..10) added by the workspace plan (stam_cuda_spadd) and by the
merge-based plan (pairwise two-way unions, stam_cuda_spadd_merge) on the GPU.
Operands: config-2 rows (200k x 200k, 50 per row) with seeds 201+p.  CSV:
k, plan, kernel_ms (sum of the call's kernels, median of 5), merge_compares,
adds, nnz."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1802_10574_b200 import Context, _native as N  # noqa: E402
from paper_1802_10574_b200 import generators as G  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
ctx = Context(0)
ops = [G.csr_fixed(rows, rows, 50, 201 + p).to("cuda") for p in range(10)]
print("k,plan,kernel_ms,merge_compares,adds,nnz")
for k in range(2, 11):
    for plan, fn in (("workspace", ctx.spadd), ("merge", ctx.spadd_merge)):
        times = []
        for rep in range(6):
            st = N.Stats()
            D = fn(ops[:k], timing=True, stats=st)
            if rep:
                times.append(st.total_kernel_ms)
        print(f"{k},{plan},{statistics.median(times):.4f},{st.merge_compares},{st.adds},{D.nnz}",
              flush=True)
        del D
