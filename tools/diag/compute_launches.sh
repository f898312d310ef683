python - <<'PY' > gpurun_out/p.log 2>&1
import sys; sys.path.insert(0,'.')
from paper_1802_10574_b200 import Context
from paper_1802_10574_b200 import generators as G
cfg=G.make_config(3); ctx=Context(0)
A=cfg['A'].to('cuda'); idx=ctx.spgemm(A,A,mode='assemble')
import torch; torch.cuda.synchronize()
C=ctx.spgemm_compute(A,A,idx); torch.cuda.synchronize(); print('ok')
PY
