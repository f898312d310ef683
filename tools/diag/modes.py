"""SpGEMM mode timings (fused / assemble / compute / unsorted) on a config,
device-resident, CUDA-event kernel sums from the library's stats."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1802_10574_b200 import Context, _native as N  # noqa: E402
from paper_1802_10574_b200 import generators as G  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = G.make_config(cid)
ctx = Context(0)
A, B = cfg["A"].to("cuda"), cfg["B"].to("cuda")


def timed(fn, reps=3):
    best = None
    for _ in range(reps + 1):
        st = N.Stats()
        out = fn(st)
        del out
        best = st.total_kernel_ms if best is None else min(best, st.total_kernel_ms)
    return best


idx = ctx.spgemm(A, B, mode="assemble")
print("fused      ms", round(timed(lambda st: ctx.spgemm(A, B, timing=True, stats=st)), 3))
print("unsorted   ms", round(timed(lambda st: ctx.spgemm(A, B, sort=False, timing=True, stats=st)), 3))
print("assemble   ms", round(timed(lambda st: ctx.spgemm(A, B, mode="assemble", timing=True, stats=st)), 3))
print("compute    ms", round(timed(lambda st: ctx.spgemm_compute(A, B, idx, timing=True, stats=st)), 3))
