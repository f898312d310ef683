"""B200-native (sm_100a) workspace sparse kernels — the engine slot of the
reference ``stam`` library (arXiv 1802.10574; ``/root/reference/proj``).

Hot path: Gustavson SpGEMM, multi-operand SpAdd and CSF MTTKRP (dense and
sparse result), each a fixed instance of the loop nest the reference's
``schedule()`` emits, run as hand-written CUDA kernels behind the C ABI in
``include/stam_cuda.h``.  This package is the Python host mirror of that
interface; the C++ mirror is ``include/stam/kernels.h``.
"""
from ._native import StamError
from .kernels import Context, default_context, mttkrp, spadd, spgemm
from .storage import CSF3, CSR, Dense

__all__ = ["StamError", "Context", "default_context", "spgemm", "spadd", "mttkrp", "CSR",
           "CSF3", "Dense"]
