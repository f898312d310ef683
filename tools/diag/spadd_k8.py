import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1802_10574_b200 import Context  # noqa: E402
from paper_1802_10574_b200 import generators as G  # noqa: E402
import torch  # noqa: E402
k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ctx = Context(0)
ops = [G.csr_fixed(200000, 200000, 50, 201 + p).to("cuda") for p in range(k)]
D = ctx.spadd(ops)
torch.cuda.synchronize()
print("ok", D.nnz)
