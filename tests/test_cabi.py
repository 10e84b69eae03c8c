"""The C-ABI library loads and exports every symbol include/axonn.h declares
(no compute calls: runs on CPU-only hosts), and the Python binding fails
loudly instead of falling back when a call cannot run."""
import ctypes as C
import os
import re
import subprocess

import pytest


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_library_builds_and_exports_all_symbols(dtype):
    """Both builds (bf16 libaxonn.so, fp16 libaxonn_fp16.so) export exactly the header's ABI
    and report their half format."""
    from paper_2110_13005_b200 import _lib, build
    build.build()
    path = build.LIBS[dtype]
    lib = C.CDLL(path, mode=C.RTLD_LOCAL)
    names = _lib.exported_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    # nothing else leaks from the shared object (hidden visibility)
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (axonn_\w+)", out))
    assert exported == set(names), exported ^ set(names)
    assert _lib.load(dtype).axonn_half_dtype() == _lib.DTYPES[dtype]


def test_dtype_mismatch_rejected_before_device():
    """axonn_model_cfg.dtype must match the library build (INVALID_ARG before any device work)."""
    from paper_2110_13005_b200 import _lib
    for dtype, other in (("bf16", 1), ("fp16", 0)):
        mc = _lib.ModelCfg(2, 64, 2, 32, 256, 42, other)
        oc = _lib.OptCfg(1e-3, 0.9, 0.999, 1e-8, 0.01, 1.0, 0, 4000000, 4, 0, 0, 0)
        ctx = C.c_void_p()
        rc = _lib.load(dtype).axonn_init(1, 1, 2, C.byref(mc), C.byref(oc), None, C.byref(ctx))
        assert rc == -1 and not ctx.value


def test_header_declares_paper_boundary():
    from paper_2110_13005_b200 import _lib
    names = set(_lib.exported_symbols())
    for n in ("axonn_init", "axonn_run_batch", "axonn_optimizer_step", "axonn_free"):
        assert n in names


def test_init_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2110_13005_b200.engine import AxoNN, AxoNNError
    with pytest.raises(AxoNNError) as e:
        AxoNN(1, 1, 1, n_layers=1, hidden=64, heads=2, seq_len=32, vocab=256)
    assert e.value.status == "CUDA"


def test_init_validation_errors_before_device():
    """Argument validation happens before any device work."""
    from paper_2110_13005_b200.engine import AxoNN, AxoNNError
    cases = [
        (dict(g_inter=2, g_data=1), dict(), "GRID_MISMATCH"),
        (dict(g_inter=1, g_data=1), dict(hidden=60), "INVALID_ARG"),
        (dict(g_inter=1, g_data=1), dict(heads=3), "INVALID_ARG"),
    ]
    for grid, over, status in cases:
        cfg = dict(n_layers=2, hidden=64, heads=2, seq_len=32, vocab=256)
        cfg.update(over)
        with pytest.raises(AxoNNError) as e:
            AxoNN(grid["g_inter"], grid["g_data"], 1, **cfg)
        assert e.value.status == status
    with pytest.raises(AxoNNError) as e:
        AxoNN(2, 1, 1, n_layers=3, hidden=64, heads=2, seq_len=32, vocab=256, world_size=2,
              nccl_id=b"x" * 128)
    assert e.value.status == "NONDIVISIBLE_LAYERS"


def test_bad_checkpoint_interval_rejected_before_device():
    """BadCheckpointInterval: ac must divide the stage's layer count."""
    from paper_2110_13005_b200.engine import AxoNN, AxoNNError
    with pytest.raises(AxoNNError) as e:
        AxoNN(1, 1, 1, n_layers=4, hidden=64, heads=2, seq_len=32, vocab=256, checkpoint_interval=3)
    assert e.value.status == "INVALID_ARG"


def _header_structs():
    """field names, in order, of every `typedef struct { ... } name;` in include/axonn.h"""
    import re
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "include", "axonn.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    hdr = re.sub(r"//[^\n]*", "", hdr)
    out = {}
    for body, name in re.findall(r"typedef struct\s*\{(.*?)\}\s*(\w+)\s*;", hdr, flags=re.S):
        fields = []
        for decl in body.split(";"):
            decl = " ".join(decl.split())
            if not decl:
                continue
            # "const double* stage_speed", "double lr, beta1", "int64_t bucket_elems"
            m = re.match(r"(?:const\s+)?[\w]+(?:\s*\*)?\s+(.*)$", decl)
            for part in m.group(1).split(","):
                fields.append(part.strip().lstrip("*").strip())
        out[name] = fields
    return out


def test_ctypes_structs_match_the_header():
    """The binding's ctypes Structures list the header's fields in the header's order (a
    missing or reordered field would shift every later one silently)."""
    from paper_2110_13005_b200 import _lib
    hs = _header_structs()
    for cname, py in (("axonn_model_cfg", _lib.ModelCfg), ("axonn_opt_cfg", _lib.OptCfg),
                      ("axonn_dist", _lib.Dist), ("axonn_gemm_args", _lib.GemmArgs)):
        assert cname in hs, (cname, list(hs))
        assert [f for f, _ in py._fields_] == hs[cname], (cname, [f for f, _ in py._fields_], hs[cname])
