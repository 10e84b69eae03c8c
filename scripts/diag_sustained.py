"""Sustained (power-capped) K1 vs cuBLAS at the 1.3B step shapes, with SM clock / power
sampled by NVML every 5 ms during each phase.  Each phase runs the same launch back to
back for ~1.5 s (no L2 flush: the operands of the real step are not L2 resident either,
but repeated launches are the sustained regime the step runs in).  Prints JSON lines."""
import ctypes as C
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class Nvml:
    def __init__(self):
        import pynvml as N
        N.nvmlInit()
        self.N = N
        self.h = N.nvmlDeviceGetHandleByIndex(int(os.environ.get("LOCAL_RANK", "0")))
        self.samples = []
        self.on = False
        self.t = threading.Thread(target=self._run, daemon=True)
        self.alive = True
        self.t.start()

    def _run(self):
        N = self.N
        while self.alive:
            if self.on:
                try:
                    self.samples.append((N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM),
                                         N.nvmlDeviceGetPowerUsage(self.h) / 1000.0))
                except Exception:
                    pass
            time.sleep(0.005)

    def start(self):
        self.samples = []
        self.on = True

    def stop(self):
        self.on = False
        s = self.samples
        if not s:
            return {}
        cl = sorted(x[0] for x in s)
        pw = sorted(x[1] for x in s)
        return {"sm_mhz_med": cl[len(cl) // 2], "sm_mhz_min": cl[0], "power_med": pw[len(pw) // 2],
                "n": len(s)}


def main():
    import torch
    from paper_2110_13005_b200 import _lib
    lib = _lib.load()
    nv = Nvml()
    st = torch.cuda.current_stream().cuda_stream
    M, h = 4096, 2048
    shapes = [("fc1 fwd gelu", "fwd", M, 4 * h, h, 1), ("fc1 fwd plain", "fwd", M, 4 * h, h, 0),
              ("fc1 dgrad", "dgrad", M, h, 4 * h, 0), ("fc2 wgrad acc", "wgrad", h, 4 * h, M, 3),
              ("fc1 wgrad acc", "wgrad", 4 * h, h, M, 3), ("qkv wgrad acc", "wgrad", 3 * h, h, M, 3),
              ("proj fwd resid", "fwd", M, h, h, 9), ("proj wgrad acc", "wgrad", h, h, M, 3)]
    only = os.environ.get("DIAG_ONLY")
    for name, kind, Mm, N, K, epi in shapes:
        if only and only not in name:
            continue
        A = torch.randn(Mm, K, device="cuda", dtype=torch.bfloat16) if kind != "wgrad" else \
            torch.randn(K, Mm, device="cuda", dtype=torch.bfloat16)
        B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) if kind == "fwd" else \
            torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
        Cb = torch.zeros(Mm, N, device="cuda", dtype=torch.float32 if kind == "wgrad" else torch.bfloat16)
        bias = torch.randn(N, device="cuda", dtype=torch.bfloat16)
        aux = torch.empty(Mm, N, device="cuda", dtype=torch.bfloat16)
        g = _lib.GemmArgs()
        g.M, g.N, g.K, g.Z, g.Z1 = Mm, N, K, 1, 1
        g.A, g.lda, g.a_mn = A.data_ptr(), (Mm if kind == "wgrad" else K), int(kind == "wgrad")
        g.B, g.ldb, g.b_mn = B.data_ptr(), (K if kind == "fwd" else N), int(kind != "fwd")
        g.C, g.ldc = Cb.data_ptr(), N
        g.alpha = 1.0
        g.variant = int(os.environ.get("DIAG_VARIANT", "0"))
        if epi == 3:
            g.epi, g.accumulate = 3, 1
        elif epi == 1:
            g.epi, g.bias, g.aux, g.ld_aux = 1, bias.data_ptr(), aux.data_ptr(), N
        elif epi == 9:
            g.epi, g.bias, g.resid, g.ld_resid = 0, bias.data_ptr(), aux.data_ptr(), N
        fl = 2.0 * Mm * N * K

        def ours():
            assert lib.axonn_k_gemm(C.byref(g), C.c_void_p(st)) == 0
        if kind == "fwd":
            ref = lambda: torch.matmul(A, B.t())
        elif kind == "dgrad":
            ref = lambda: torch.matmul(A, B)
        else:
            ref = lambda: torch.matmul(A.t(), B)
        res = {"shape": name, "M": Mm, "N": N, "K": K}
        for tag, fn in (("ours", ours), ("cublas", ref)):
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            # one burst launch (cool GPU) then a sustained loop
            time.sleep(0.3)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            burst = e0.elapsed_time(e1)
            n = max(20, int(1500 / max(burst, 1e-3)))
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
            nv.start()
            evs[0].record()
            for i in range(n):
                fn()
                evs[i + 1].record()
            torch.cuda.synchronize()
            clk = nv.stop()
            ts = [evs[i].elapsed_time(evs[i + 1]) for i in range(n)]
            tail = sorted(ts[n // 2:])
            med = tail[len(tail) // 2]
            res[tag] = {"burst_tflops": fl / burst / 1e9, "sustained_tflops": fl / med / 1e9,
                        "sustained_us": med * 1e3, "launches": n, **clk}
        print(json.dumps(res), flush=True)
        del A, B, Cb, aux
        torch.cuda.empty_cache()
        time.sleep(0.5)
    nv.alive = False


if __name__ == "__main__":
    main()
