"""PCIe diagnostics: H2D / D2H / duplex bandwidth and the SpAdd call with
host inputs and/or host result (config 2)."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

from paper_1802_10574_b200 import Context, _native as N  # noqa: E402
from paper_1802_10574_b200 import generators as G  # noqa: E402


def bw(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    return nbytes / dt / 1e9, dt * 1e3


n = 60_000_000  # 480 MB of f64
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
print("h2d GB/s, ms", bw(lambda: d.copy_(h, non_blocking=True), n * 8))
print("d2h GB/s, ms", bw(lambda: h2.copy_(d2, non_blocking=True), n * 8))


def duplex():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


print("duplex GB/s (both dirs), ms", bw(duplex, 2 * n * 8))
# kernel writing to mapped host memory
hm = h2
print("kernel copy d->mapped host GB/s, ms",
      bw(lambda: torch.ops.aten.copy_(hm, d, True), n * 8))

cfg = G.make_config(2)
ctx = Context(0)
lib = N.load()
dev = [o.to("cuda") for o in cfg["ops"]]
dviews = (N.CsrView * 3)(*[o.view() for o in dev])
pinned = [[torch.from_numpy(a).pin_memory() for a in (o.pos, o.idx, o.vals)] for o in cfg["ops"]]
from paper_1802_10574_b200.storage import CSR  # noqa: E402

hops = [CSR(o.nrows, o.ncols, *arrs) for o, arrs in zip(cfg["ops"], pinned)]
hviews = (N.CsrView * 3)(*[x.view() for x in hops])
for v in hviews:
    v.mem = N.STAM_MEM_HOST


def call(views, rmem):
    r = N.CsrResult()
    st = N.Stats()
    opts = N.Options(1, 0, rmem, 0)
    N.check(lib.stam_cuda_spadd(ctx._ctx, 3, views, C.byref(opts), C.byref(r), C.byref(st)))
    N.check(lib.stam_cuda_release(ctx._ctx, C.c_void_p(r.handle)))


for name, views, rmem in [("dev->dev", dviews, N.STAM_MEM_DEVICE),
                          ("host->dev", hviews, N.STAM_MEM_DEVICE),
                          ("dev->host", dviews, N.STAM_MEM_HOST),
                          ("host->host", hviews, N.STAM_MEM_HOST)]:
    print(name, "ms", bw(lambda: call(views, rmem), 1)[1])
