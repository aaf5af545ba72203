"""B200-native (sm_100a) hot path of arXiv 2405.09400 — entropic domain
decomposition sweeps with flow updates, as a C-ABI CUDA library
(libdomdec.so, include/domdec.h) plus this thin ctypes binding.

PyTorch is optional plumbing (streams, device memory for benchmarks,
torch.distributed for multi-process runs); the computation is entirely in the
library's CUDA kernels.  There is no CPU fallback.
"""
from ._lib import (DomDec, DomDecError, FlowStats, SweepStats, mincost_flow, mufu_peak, lib, sinkhorn_global,  # noqa: F401,E501
                   multiscale_solve,
                   LIB_PATH, EXPORTED, PART_A, PART_B)
from .build import build_library  # noqa: F401
