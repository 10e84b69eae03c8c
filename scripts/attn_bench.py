"""Time the fused attention kernels at the 1.3B / 12B attention shapes (µs per launch)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2110_13005_b200 import _lib
    if "--lib" in sys.argv:   # a diagnostic build (paper_2110_13005_b200/build.py AXONN_DIAG_TAG)
        lib = _lib._declare(C.CDLL(sys.argv[sys.argv.index("--lib") + 1]))
    else:
        lib = _lib.load()
    tag_arg = sys.argv[sys.argv.index("--tag") + 1] if "--tag" in sys.argv else ""
    bs = int(sys.argv[sys.argv.index("--b") + 1]) if "--b" in sys.argv else 8
    st = torch.cuda.current_stream().cuda_stream
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    for tag, b, heads, s, d, dp in (("1.3B", bs, 16, 512, 128, 128), ("12B", bs, 24, 512, 188, 192)):
        if only and tag != only:
            continue
        lq = 3 * heads * dp
        qkv = (torch.randn(b * s, lq, device="cuda") * 0.5).to(torch.bfloat16)
        o = torch.empty(b * s, heads * d, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(b * heads * s, device="cuda", dtype=torch.float32)
        alpha = 1.0 / d ** 0.5

        def fwd():
            assert lib.axonn_k_attn_fwd(C.c_void_p(qkv.data_ptr()), lq, b, heads, s, d, dp, C.c_float(alpha),
                                        C.c_void_p(o.data_ptr()), heads * d, C.c_void_p(lse.data_ptr()),
                                        C.c_void_p(st)) == 0
        for _ in range(1 if only else 5):
            fwd()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 3 if only else 50
        e0.record()
        for _ in range(n):
            fwd()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / n * 1e3
        fl = 4.0 * b * heads * s * s * dp / 2   # causal half of QK^T and PV
        print(json.dumps({"kernel": "attn_fwd", "shape": tag, "b": b, "variant": tag_arg, "us": us,
                          "tflops_causal": fl / us / 1e6}),
              flush=True)
        dO = (torch.randn(b * s, heads * dp, device="cuda") * 0.1).to(torch.bfloat16)
        dbuf = torch.empty(b * heads * s, device="cuda", dtype=torch.float32)
        dqkv = torch.empty(b * s, 3 * heads * d, device="cuda", dtype=torch.bfloat16)

        def bwd():
            P = C.c_void_p
            assert lib.axonn_k_attn_bwd(P(qkv.data_ptr()), lq, P(dO.data_ptr()), P(o.data_ptr()), heads * d,
                                        P(lse.data_ptr()), P(dbuf.data_ptr()), b, heads, s, d, dp,
                                        C.c_float(alpha), P(dqkv.data_ptr()), 3 * heads * d, P(st)) == 0
        for _ in range(1 if only else 5):
            bwd()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(n):
            bwd()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / n * 1e3
        print(json.dumps({"kernel": "attn_bwd", "shape": tag, "b": b, "variant": tag_arg, "us": us,
                          "tflops_causal": 2.5 * fl / us / 1e6}), flush=True)


if __name__ == "__main__":
    main()
