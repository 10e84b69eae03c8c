"""Build the C-ABI libraries in-tree: every .cu / .cpp under csrc/ compiled for sm_100a
with nvcc (one process per source file, in parallel), linked against the torch-bundled
NCCL 2.28 (same libnccl.so.2 that torch loads, so one NCCL runtime per process).

Two builds of the same sources, one per half-precision format (include/axonn.h
axonn_dtype; csrc/half.cuh):
  libaxonn.so       bf16 (reading D-31, the default)
  libaxonn_fp16.so  fp16 (-DAXONN_HALF_FP16; the paper's format with loss scaling, §8(f) N2)
The oracle is pure numpy: nothing to compile."""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
LIBS = {"bf16": os.path.join(HERE, "libaxonn.so"), "fp16": os.path.join(HERE, "libaxonn_fp16.so")}
# diagnostic builds only (never loaded by the package): extra -D defines into a separately
# named library, e.g. AXONN_DIAG_DEFINES="-DAXONN_ATTN_EXP=1" AXONN_DIAG_TAG=_exp1
DIAG_DEFINES = os.environ.get("AXONN_DIAG_DEFINES", "").split()
DIAG_TAG = os.environ.get("AXONN_DIAG_TAG", "")
if DIAG_TAG:
    LIBS = {k: v.replace(".so", DIAG_TAG + ".so") for k, v in LIBS.items()}
LIB = LIBS["bf16"]
DEFINES = {"bf16": [], "fp16": ["-DAXONN_HALF_FP16"]}


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        inc = os.path.join(base, "nccl", "include")
        lib = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("NCCL headers (nvidia-nccl wheel) not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _digest(dtype: str):
    h = hashlib.sha256((dtype + " ".join(DIAG_DEFINES)).encode())
    for f in sources() + sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))) + [
            os.path.join(ROOT, "include", "axonn.h"), __file__]:
        with open(f, "rb") as fh:
            h.update(f.encode() + fh.read())
    return h.hexdigest()


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    return r.returncode, r.stdout + r.stderr


def _build_one(dtype: str, force: bool, verbose: bool, pool: ThreadPoolExecutor) -> str:
    lib_path = LIBS[dtype]
    stamp = lib_path + ".sha"
    dig = _digest(dtype)
    if not force and os.path.exists(lib_path) and os.path.exists(stamp) and open(stamp).read() == dig:
        return lib_path
    inc, lib = nccl_dirs()
    objdir = os.path.join(HERE, "build", dtype + DIAG_TAG)
    os.makedirs(objdir, exist_ok=True)
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
             "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
             "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc] + DEFINES[dtype] + DIAG_DEFINES
    if verbose:
        flags = ["-Xptxas=-v"] + flags
    objs, jobs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        jobs.append(pool.submit(_run, [NVCC] + flags + ["-c", src, "-o", obj]))
    for src, j in zip(sources(), jobs):
        rc, out = j.result()
        if rc != 0 or verbose:
            sys.stderr.write(out)
        if rc != 0:
            raise RuntimeError(f"nvcc failed on {os.path.basename(src)} ({dtype})")
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib_path + ".tmp"] + objs + [
        "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib, "-Xlinker", "-Bsymbolic", "-lcudart"]
    rc, out = _run(link)
    if rc != 0:
        sys.stderr.write(out)
        raise RuntimeError(f"nvcc link failed ({dtype})")
    os.replace(lib_path + ".tmp", lib_path)
    with open(stamp, "w") as f:
        f.write(dig)
    return lib_path


def build(force: bool = False, verbose: bool = False, dtypes=("bf16", "fp16")) -> str:
    """Build (if stale) every library in ``dtypes``; returns the bf16 library path."""
    with ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as pool:
        paths = [_build_one(d, force, verbose, pool) for d in dtypes]
    return LIB if "bf16" in dtypes else paths[0]


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
