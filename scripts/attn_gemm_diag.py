"""Why are the batched attention products (P V, dS K, dS^T Q, P^T dO at b 8 x 16 heads,
s 512, d 128) slow?  Times variants of the P V launch: as in the step, without the causal
range, with a contiguous output, unbatched, and under the AXONN_GEMM_DBG experiments
(set by the caller).  One JSON line per variant (µs per launch, back-to-back)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2110_13005_b200 import _lib
    lib = _lib.load()
    b, a, s, d = 8, 16, 512, 128
    h = a * d
    st = torch.cuda.current_stream().cuda_stream
    qkv = (torch.randn(b * s, 3 * h, device="cuda") * 0.5).to(torch.bfloat16)
    P = (torch.rand(b, a, s, s, device="cuda") * 0.01).to(torch.bfloat16)
    o = torch.empty(b * s, h, device="cuda", dtype=torch.bfloat16)
    oc = torch.empty(b * a, s, d, device="cuda", dtype=torch.bfloat16)
    big = torch.empty(b * a * s, s, device="cuda", dtype=torch.bfloat16)

    def pv(causal=2, contiguous=False, variant=0):
        g = _lib.GemmArgs()
        g.M, g.N, g.K, g.Z, g.Z1 = s, d, s, b * a, a
        g.n_valid = d
        g.A, g.lda, g.a_s1, g.a_s2 = P.data_ptr(), s, s * s, a * s * s
        g.B, g.ldb, g.b_s1, g.b_s2, g.b_mn = qkv.data_ptr() + 2 * h * 2, 3 * h, d, s * 3 * h, 1
        if contiguous:
            g.C, g.ldc, g.c_s1, g.c_s2 = oc.data_ptr(), d, s * d, a * s * d
        else:
            g.C, g.ldc, g.c_s1, g.c_s2 = o.data_ptr(), h, d, s * h
        g.epi, g.causal, g.alpha, g.variant = 0, causal, 1.0, variant
        return g

    def flat():
        # unbatched: [b*a*s, s] x [s, d] (B = first 512 rows of V, MN-major), same FLOPs as non-causal
        g = _lib.GemmArgs()
        g.M, g.N, g.K, g.Z, g.Z1 = b * a * s, d, s, 1, 1
        g.A, g.lda = P.data_ptr(), s
        g.B, g.ldb, g.b_mn = qkv.data_ptr() + 2 * h * 2, 3 * h, 1
        g.C, g.ldc = oc.data_ptr(), d
        g.epi, g.alpha = 0, 1.0
        return g

    def timeit(g, n=50):
        for _ in range(5):
            assert lib.axonn_k_gemm(C.byref(g), C.c_void_p(st)) == 0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            lib.axonn_k_gemm(C.byref(g), C.c_void_p(st))
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n * 1e3

    dbg = os.environ.get("AXONN_GEMM_DBG", "0")
    for name, g in [("pv step (causal2, merged heads)", pv()), ("pv causal0", pv(causal=0)),
                    ("pv contiguous out", pv(contiguous=True)),
                    ("pv pair variant2", pv(variant=2)),
                    ("flat 65536x128x512", flat())]:
        print(json.dumps({"dbg": dbg, "case": name, "us": timeit(g)}), flush=True)
    del big


if __name__ == "__main__":
    main()
