"""B200-native AxoNN hybrid training step (arXiv 2110.13005).

The product is the C-ABI shared library ``libaxonn.so`` (include/axonn.h):
hand-written sm_100a kernels (tcgen05/TMEM/TMA GEMMs, warp-shuffle LayerNorm /
softmax / cross-entropy, fused AdamW), a message-driven per-stage scheduler
on CUDA streams and events, NCCL P2P and all-reduce over NVLink, and the
bucketed pinned-host optimizer.  This package is a thin binding:
``_lib`` (ctypes marshalling), ``engine`` (Python wrapper of a context) and
``dist`` (torch.distributed bootstrap of the NCCL unique id)."""
from ._lib import load  # noqa: F401
