import ctypes as C, os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
from paper_1802_10574_b200 import Context, _native as N
from paper_1802_10574_b200 import generators as G
from paper_1802_10574_b200.storage import CSR
cfg = G.make_config(2); ctx = Context(0); lib = N.load()
pinned = [[torch.from_numpy(a).pin_memory() for a in (o.pos, o.idx, o.vals)] for o in cfg["ops"]]
hops = [CSR(o.nrows, o.ncols, *arrs) for o, arrs in zip(cfg["ops"], pinned)]
hviews = (N.CsrView * 3)(*[x.view() for x in hops])
for v in hviews: v.mem = N.STAM_MEM_HOST
def call():
    r = N.CsrResult(); st = N.Stats(); opts = N.Options(1, 0, N.STAM_MEM_HOST, 0)
    N.check(lib.stam_cuda_spadd(ctx._ctx, 3, hviews, C.byref(opts), C.byref(r), C.byref(st)))
    N.check(lib.stam_cuda_release(ctx._ctx, C.c_void_p(r.handle)))
call(); call()
os.environ["STAM_DEBUG_STREAM"] = "1"
t = time.perf_counter(); call(); print("total ms", (time.perf_counter() - t) * 1e3, flush=True)
