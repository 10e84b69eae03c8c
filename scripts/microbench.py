"""Kernel sweeps of BASELINE.json configs[4] / SURVEY.md §8(d) D4.

(i)  K1 GEMM at every per-layer shape of the 1.3B / 12B / 24B configs (fwd, dgrad,
     wgrad layouts) and the LM head, TFLOP/s of our tcgen05 kernel (single-CTA and
     CTA-pair variants) beside cuBLAS (torch.matmul, the vendor yardstick) at the
     same shape and operand layout.
(iii) K9 AdamW in HBM (28 B/param) and the engine's bucketed offload step
     (12 B/param each way over the host link) for several bucket sizes.
Writes one JSON object per line to stdout."""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def time_cuda(fn, iters=10, warm=3):
    import torch
    st = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tot = 0.0
    for _ in range(iters):
        flush.zero_()   # > L2 between timed launches
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        tot += a.elapsed_time(b)
    return tot / iters


def gemm_sweep(variants=(0, 1, 2), only=None, iters=10):
    import torch
    from paper_2110_13005_b200 import _lib
    lib = _lib.load()
    shapes = []
    for tag, M, h in (("1.3B", 4096, 2048), ("12B", 4096, 4512), ("24B", 2048, 6336)):
        for name, N, K in (("qkv", 3 * h, h), ("proj", h, h), ("fc1", 4 * h, h), ("fc2", h, 4 * h)):
            shapes.append((tag, name, "fwd", M, N, K))
            shapes.append((tag, name, "dgrad", M, K, N))
            shapes.append((tag, name, "wgrad", N, K, M))
        shapes.append((tag, "head", "fwd", M, 51200, h))
    out = []
    if only:
        shapes = [s for s in shapes if f"{s[0]} {s[1]} {s[2]}" == only]
    for tag, name, kind, M, N, K in shapes:
        # operands in the layouts the step uses
        A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16) if kind != "wgrad" else \
            torch.randn(K, M, device="cuda", dtype=torch.bfloat16)
        B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) if kind == "fwd" else \
            torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
        Cb = torch.empty(M, N, device="cuda", dtype=torch.float32 if kind == "wgrad" else torch.bfloat16)
        st = torch.cuda.current_stream().cuda_stream
        res = {"shape": f"{tag} {name} {kind}", "M": M, "N": N, "K": K}
        fl = 2.0 * M * N * K
        for v in variants:
            g = _lib.GemmArgs()
            g.M, g.N, g.K, g.Z, g.Z1 = M, N, K, 1, 1
            g.A, g.lda, g.a_mn = A.data_ptr(), (M if kind == "wgrad" else K), int(kind == "wgrad")
            g.B, g.ldb, g.b_mn = B.data_ptr(), (K if kind == "fwd" else N), int(kind != "fwd")
            g.C, g.ldc = Cb.data_ptr(), N
            g.epi = 3 if kind == "wgrad" else 0
            g.accumulate = 1 if kind == "wgrad" else 0
            g.alpha = 1.0
            g.variant = v

            def run(g=g):
                rc = lib.axonn_k_gemm(C.byref(g), C.c_void_p(st))
                assert rc == 0, rc
            ms = time_cuda(run, iters=iters, warm=min(3, iters))
            res[f"ours_v{v}_tflops"] = fl / ms / 1e9
        if kind == "fwd":
            ref = lambda: torch.matmul(A, B.t())
        elif kind == "dgrad":
            ref = lambda: torch.matmul(A, B)
        else:
            ref = lambda: torch.matmul(A.t(), B)
        res["cublas_tflops"] = fl / time_cuda(ref, iters=iters, warm=min(3, iters)) / 1e9
        if kind == "fwd" and name in ("fc1", "proj"):   # the step's fused epilogues
            bias = torch.randn(N, device="cuda", dtype=torch.bfloat16)
            aux = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            g = _lib.GemmArgs()
            g.M, g.N, g.K, g.Z, g.Z1 = M, N, K, 1, 1
            g.A, g.lda, g.B, g.ldb, g.C, g.ldc = A.data_ptr(), K, B.data_ptr(), K, Cb.data_ptr(), N
            g.alpha, g.bias = 1.0, bias.data_ptr()
            if name == "fc1":
                g.epi, g.aux, g.ld_aux = 1, aux.data_ptr(), N        # bias + GeLU (+ pre store)
            else:
                g.epi, g.resid, g.ld_resid = 0, aux.data_ptr(), N    # bias + residual
            res["ours_fused_epilogue_tflops"] = fl / time_cuda(
                lambda: lib.axonn_k_gemm(C.byref(g), C.c_void_p(st))) / 1e9
        if kind == "dgrad" and name == "fc2":   # dgrad with GeLU' of the stored pre-activation
            aux = torch.randn(M, N, device="cuda", dtype=torch.bfloat16)
            g = _lib.GemmArgs()
            g.M, g.N, g.K, g.Z, g.Z1 = M, N, K, 1, 1
            g.A, g.lda, g.B, g.ldb, g.b_mn = A.data_ptr(), K, B.data_ptr(), N, 1
            g.C, g.ldc, g.alpha = Cb.data_ptr(), N, 1.0
            g.epi, g.aux, g.ld_aux = 2, aux.data_ptr(), N
            res["ours_fused_epilogue_tflops"] = fl / time_cuda(
                lambda: lib.axonn_k_gemm(C.byref(g), C.c_void_p(st))) / 1e9
        out.append(res)
        print(json.dumps(res), flush=True)
        del A, B, Cb
    return out


def host_link_probe():
    """Pinned host <-> HBM copy bandwidth (the offloaded optimizer's roofline, SURVEY.md
    §8(d.3) A7): H2D alone, D2H alone, and both directions at once on two streams."""
    import torch
    n = 1 << 30
    h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, pairs in (("h2d", [(d1, h1, s1)]), ("d2h", [(h2, d2, s2)]),
                        ("duplex", [(d1, h1, s1), (h2, d2, s2)])):
        best = 0.0
        for _ in range(3):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for dst, src, st in pairs:
                st.wait_event(e0)
                with torch.cuda.stream(st):
                    dst.copy_(src, non_blocking=True)
            for _, _, st in pairs:
                torch.cuda.current_stream().wait_stream(st)
            e1.record()
            torch.cuda.synchronize()
            gbs = len(pairs) * n / (e0.elapsed_time(e1) / 1e3) / 1e9
            best = max(best, gbs)
        res[name + "_GBps"] = best
    r = {"kernel": "host link probe (pinned, 1 GiB)", **res}
    print(json.dumps(r), flush=True)
    return res


def adam_sweep():
    import torch
    from paper_2110_13005_b200 import _lib
    lib = _lib.load()
    n = 1 << 28
    th = torch.randn(n, device="cuda") * 0.02
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    g = (torch.randn(n, device="cuda") * 1e-3).to(torch.bfloat16)
    t16 = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    sc = (C.c_float * 9)(*[1 - 1e-5, 0.9, 0.1, 0.999, 0.001, 1e-2, 0.0447, 1e-8, 1.0])
    st = torch.cuda.current_stream().cuda_stream

    def run():
        assert lib.axonn_k_adamw(n, g.data_ptr(), th.data_ptr(), m.data_ptr(), v.data_ptr(),
                                 t16.data_ptr(), sc, C.c_void_p(st)) == 0
    ms = time_cuda(run, iters=5)
    r = {"kernel": "K9 adamw in HBM", "params": n, "ms": ms, "GB/s": 28.0 * n / ms / 1e6}
    print(json.dumps(r), flush=True)
    del th, m, v, g, t16
    torch.cuda.empty_cache()
    probe = host_link_probe()
    # engine-level offloaded optimizer step (pinned host theta/m/v, 3-slot ring)
    from paper_2110_13005_b200.engine import AxoNN
    from synth import uniform_tokens
    for bs in (1 << 20, 4_000_000, 16_000_000, 64_000_000):
        for off in (1, 0):
            eng = AxoNN(1, 1, 1, n_layers=2, hidden=2048, heads=16, seq_len=512, vocab=51200,
                        offload=bool(off), bucket_elems=bs, coarsen_k=4, overlap_next_batch=False)
            phi = sum(t[2] for t in eng.tensors())
            tok = uniform_tokens(1, 512, 51200)
            ts = []
            for it in range(4):
                eng.run_batch(tok)
                eng.optimizer_step()
                ts.append(eng.stats()["t_opt_ms"])
            ms = float(np.median(ts[1:]))
            per = 24.0 if off else 28.0
            r = {"kernel": "optimizer_step " + ("offload" if off else "in-HBM"), "bucket": bs,
                 "params": phi, "ms": ms, "GB/s": per * phi / ms / 1e6,
                 "bytes_per_param": per}
            if off and probe:
                r["frac_of_duplex_probe"] = per * phi / ms / 1e6 / probe["duplex_GBps"]
            print(json.dumps(r), flush=True)
            eng.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="gemm,adam")
    ap.add_argument("--only", default=None, help='one shape, e.g. "1.3B fc1 fwd"')
    ap.add_argument("--variants", default="0,1,2")
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    if "gemm" in a.what:
        gemm_sweep(tuple(int(v) for v in a.variants.split(",")), a.only, a.iters)
    if "adam" in a.what:
        adam_sweep()
