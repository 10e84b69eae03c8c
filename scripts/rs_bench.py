"""Time the attention-score GEMM variants at the 1.3B shape (b 8, heads 16, s 512, d 128):
fused row-softmax epilogue (AXONN_RS_DEBUG experiments 0/2/3/4) vs the fp32-output GEMM."""
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
    qkv = (torch.randn(b * s, 3 * h, device="cuda") * 0.5).to(torch.bfloat16)
    P = torch.empty(b, a, s, s, device="cuda", dtype=torch.bfloat16)
    S = torch.empty(b, a, s, s, device="cuda", dtype=torch.float32)
    st = torch.cuda.current_stream().cuda_stream

    def args(epi, C_):
        g = _lib.GemmArgs()
        g.M, g.N, g.K, g.Z, g.Z1 = s, s, d, b * a, a
        g.A, g.lda, g.a_s1, g.a_s2 = qkv.data_ptr(), 3 * h, d, s * 3 * h
        g.B, g.ldb, g.b_s1, g.b_s2 = qkv.data_ptr() + h * 2, 3 * h, d, s * 3 * h
        g.C, g.ldc, g.c_s1, g.c_s2 = C_.data_ptr(), s, s * s, a * s * s
        g.epi, g.causal, g.alpha = epi, 1, 1.0 / d ** 0.5
        return g

    def timeit(g, n=20):
        for _ in range(3):
            assert lib.axonn_k_gemm(C.byref(g), C.c_void_p(st)) == 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            lib.axonn_k_gemm(C.byref(g), C.c_void_p(st))
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / n * 1e3

    out = {}
    for dbg in ("0", "2", "3", "4", "5", "6"):
        os.environ["AXONN_RS_DEBUG"] = dbg
        out[f"rowsoftmax dbg{dbg} us"] = timeit(args(4, P))
    os.environ["AXONN_RS_DEBUG"] = "0"
    out["scores fp32 GEMM (unfused) us"] = timeit(args(3, S))
    # fixed per-launch cost: one-tile GEMMs
    A1 = torch.randn(256, 64, device="cuda").to(torch.bfloat16)
    C1 = torch.empty(256, 256, device="cuda", dtype=torch.bfloat16)
    for var in (1, 2):
        g = _lib.GemmArgs()
        g.M, g.N, g.K, g.Z, g.Z1 = 256 if var == 2 else 128, 256, 64, 1, 1
        g.A, g.lda, g.B, g.ldb, g.C, g.ldc = A1.data_ptr(), 64, A1.data_ptr(), 64, C1.data_ptr(), 256
        g.alpha, g.variant = 1.0, var
        out[f"one-tile gemm variant{var} us"] = timeit(g, 50)
    # the narrow attention product P V at the 1.3B shape
    O = torch.empty(b * s, h, device="cuda", dtype=torch.bfloat16)
    g = _lib.GemmArgs()
    g.M, g.N, g.K, g.Z, g.Z1 = s, d, s, b * a, a
    g.A, g.lda, g.a_s1, g.a_s2 = P.data_ptr(), s, s * s, a * s * s
    g.B, g.ldb, g.b_s1, g.b_s2, g.b_mn = qkv.data_ptr() + 2 * h * 2, 3 * h, d, s * 3 * h, 1
    g.C, g.ldc, g.c_s1, g.c_s2 = O.data_ptr(), h, d, s * h
    g.causal, g.alpha = 2, 1.0
    out["PV gemm us"] = timeit(g)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
