"""B200-native AxoNN hybrid training step (arXiv 2110.13005).

The product is the C-ABI shared library ``libaxonn.so`` (include/axonn.h):
hand-written sm_100a kernels (tcgen05/TMEM/TMA GEMMs, warp-shuffle LayerNorm /
softmax / cross-entropy, fused AdamW), a message-driven per-stage scheduler
on CUDA streams and events, NCCL P2P and all-reduce over NVLink, and the
bucketed pinned-host optimizer.  This package is a thin binding:
``_lib`` (ctypes marshalling), ``engine`` (Python wrapper of a context) and
``dist`` (torch.distributed bootstrap of the NCCL unique id)."""
import os as _os

# Alg. 2 pre-posts receives: a pending ncclRecv kernel spins until its
# message lands.  With more streams than CUDA hardware work queues (default 8) a later
# kernel of another stream can be queued behind it and never start.  Give every
# library stream its own queue; must be set before the process creates its CUDA context.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# libaxonn force-loads its kernels in axonn_init; eager loading also covers torch's.
_os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

from ._lib import load  # noqa: E402,F401
