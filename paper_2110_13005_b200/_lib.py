"""ctypes binding of libaxonn.so / libaxonn_fp16.so (include/axonn.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; there is
no Python or CPU fallback.  If the shared library is missing or cannot be
loaded this module raises immediately."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libaxonn.so")
LIB_PATHS = {"bf16": LIB_PATH, "fp16": os.path.join(HERE, "libaxonn_fp16.so")}
DTYPES = {"bf16": 0, "fp16": 1}   # axonn_dtype

_libs: dict = {}


class GemmArgs(C.Structure):
    _fields_ = [("M", C.c_int), ("N", C.c_int), ("K", C.c_int), ("Z", C.c_int), ("Z1", C.c_int),
                ("A", C.c_void_p), ("lda", C.c_int64), ("a_s1", C.c_int64), ("a_s2", C.c_int64),
                ("a_mn", C.c_int),
                ("B", C.c_void_p), ("ldb", C.c_int64), ("b_s1", C.c_int64), ("b_s2", C.c_int64),
                ("b_mn", C.c_int),
                ("C", C.c_void_p), ("ldc", C.c_int64), ("c_s1", C.c_int64), ("c_s2", C.c_int64),
                ("epi", C.c_int), ("causal", C.c_int), ("accumulate", C.c_int),
                ("col_group_in", C.c_int), ("col_group_out", C.c_int), ("n_valid", C.c_int),
                ("bias", C.c_void_p), ("resid", C.c_void_p), ("ld_resid", C.c_int64),
                ("aux", C.c_void_p), ("ld_aux", C.c_int64),
                ("alpha", C.c_float), ("max_ctas", C.c_int), ("variant", C.c_int)]


class ModelCfg(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("hidden", C.c_int), ("heads", C.c_int),
                ("seq_len", C.c_int), ("vocab", C.c_int), ("init_seed", C.c_uint64),
                ("dtype", C.c_int)]


class OptCfg(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("weight_decay", C.c_double), ("loss_scale", C.c_double),
                ("offload", C.c_int),
                ("bucket_elems", C.c_int64), ("coarsen_k", C.c_int), ("pipeline_limit", C.c_int),
                ("checkpoint_interval", C.c_int), ("overlap_next_batch", C.c_int),
                ("stage_balance", C.c_int), ("stage_speed", C.POINTER(C.c_double)),
                ("grad_accum_fp32", C.c_int)]


class Dist(C.Structure):
    _fields_ = [("world_rank", C.c_int), ("world_size", C.c_int), ("nccl_id", C.c_void_p),
                ("device", C.c_int), ("local_group", C.c_void_p)]


def _declare(lib):
    P, I, I64, F = C.c_void_p, C.c_int, C.c_int64, C.c_float
    sig = {
        "axonn_half_dtype": (I, []),
        "axonn_get_unique_id": (I, [P]),
        "axonn_init": (I, [I, I, I, C.POINTER(ModelCfg), C.POINTER(OptCfg), C.POINTER(Dist),
                           C.POINTER(C.c_void_p)]),
        "axonn_run_batch": (I, [P, P, I, C.POINTER(F)]),
        "axonn_run_batch_device": (I, [P, P, I, C.POINTER(F)]),
        "axonn_optimizer_step": (I, [P]),
        "axonn_free": (None, [P]),
        "axonn_last_error": (C.c_char_p, [P]),
        "axonn_num_tensors": (I, [P]),
        "axonn_tensor_info": (I, [P, I, C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "axonn_read_tensor": (I, [P, I, I, P]),
        "axonn_write_tensor": (I, [P, I, I, P]),
        "axonn_stats": (I, [P, C.POINTER(C.c_double), I]),
        "axonn_set_profiling": (I, [P, I]),
        "axonn_profile_json": (I, [P, C.c_char_p, I]),
        "axonn_timer_mark": (I, [P, I]),
        "axonn_timer_elapsed": (I, [P, I, I, C.POINTER(C.c_double)]),
        "axonn_stage_partition": (I, [C.POINTER(ModelCfg), I, C.POINTER(C.c_double), C.POINTER(I)]),
        "axonn_calibrate_speed": (I, [I, I, I, I, I, C.POINTER(C.c_double)]),
        "axonn_local_group_create": (I, [I, C.POINTER(C.c_void_p)]),
        "axonn_local_group_free": (None, [P]),
        "axonn_checkpoint_interval": (I, [P]),
        "axonn_k_gemm": (I, [C.POINTER(GemmArgs), P]),
        "axonn_k_adamw": (I, [I64, P, P, P, P, P, C.POINTER(F), P]),
        "axonn_k_attn_fwd": (I, [P, I64, I, I, I, I, I, F, P, I64, P, P]),
        "axonn_k_attn_bwd": (I, [P, I64, P, P, I64, P, P, I, I, I, I, I, F, P, I64, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    return lib


def load(dtype: str = "bf16"):
    """Load (building first if needed) the in-tree library of the half format ``dtype``
    ('bf16' -> libaxonn.so, 'fp16' -> libaxonn_fp16.so).  Both export the same symbols, so
    the fp16 build is opened RTLD_LOCAL (and both are linked -Bsymbolic)."""
    if dtype not in LIB_PATHS:
        raise ValueError(f"dtype must be one of {list(LIB_PATHS)}")
    if dtype not in _libs:
        path = LIB_PATHS[dtype]
        if not os.path.exists(path):
            from . import build
            build.build(dtypes=(dtype,))
        lib = _declare(C.CDLL(path, mode=C.RTLD_GLOBAL if dtype == "bf16" else C.RTLD_LOCAL))
        if lib.axonn_half_dtype() != DTYPES[dtype]:
            raise RuntimeError(f"{path} reports half format {lib.axonn_half_dtype()}, expected {dtype}")
        _libs[dtype] = lib
    return _libs[dtype]


def exported_symbols():
    """Names declared with AXONN_API in include/axonn.h."""
    import re
    hdr = os.path.join(os.path.dirname(HERE), "include", "axonn.h")
    return re.findall(r"AXONN_API\s+[\w\s\*]+?\b(axonn_\w+)\(", open(hdr).read())
