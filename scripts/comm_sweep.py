"""SURVEY.md §8(d) D4 (ii) and the all-reduce sweep: NVLink GB/s of the transport the
library's Alg. 2 Send/Receive and column all-reduce use (NCCL 2.28 P2P / AllReduce over
NVLink 5 / NVSwitch), at the paper's message sizes ("1-50 MB"; 16.78 MB
= 1.3B activation, 25.95 MB = 24B, 36.96 MB = 12B message) and the all-reduce chunk sizes
(k * bsize = 16 M bf16 elements = 32 MB).  Also the cudaMemcpyPeerAsync
probe.  Timing: CUDA events on the issuing stream after warm-up, max over ranks.

Run: torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/comm_sweep.py"""
import json
import os

import torch
import torch.distributed as dist

MB = 1 << 20


def timed(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = []
    sizes = [1, 2, 4, 8, 16, 16.78, 25.95, 32, 36.96, 50, 64]
    peer = rank ^ 1
    if world >= 2 and peer < world:
        for mb in sizes:
            n = int(mb * MB) // 2
            x = torch.randn(n, device="cuda").to(torch.bfloat16)
            y = torch.empty_like(x)

            def uni():
                if rank % 2 == 0:
                    dist.send(x, peer)
                else:
                    dist.recv(y, peer)

            def bi():
                ops = [dist.P2POp(dist.isend, x, peer), dist.P2POp(dist.irecv, y, peer)]
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
            ms_u = timed(uni)
            ms_b = timed(bi)
            out.append({"kind": "p2p", "MB": mb, "bytes": n * 2, "uni_ms": ms_u,
                        "uni_GBps": n * 2 / ms_u / 1e6, "bidir_ms": ms_b,
                        "bidir_GBps_per_dir": n * 2 / ms_b / 1e6})
    for mb in (8, 32, 128, 512):
        n = mb * MB // 2
        x = torch.randn(n, device="cuda").to(torch.bfloat16)
        ms = timed(lambda: dist.all_reduce(x))
        alg = n * 2 / ms / 1e6
        out.append({"kind": "allreduce_bf16", "world": world, "MB": mb, "ms": ms, "algbw_GBps": alg,
                    "busbw_GBps": alg * 2 * (world - 1) / world})
    if rank == 0 and torch.cuda.device_count() > 1:
        for mb in (16, 64):
            n = mb * MB
            a = torch.empty(n, dtype=torch.uint8, device="cuda:0")
            b = torch.empty(n, dtype=torch.uint8, device="cuda:1")
            for _ in range(3):
                b.copy_(a)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                b.copy_(a)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            out.append({"kind": "memcpy_peer", "MB": mb, "ms": ms, "GBps": n / ms / 1e6})
    if rank == 0:
        for r in out:
            print(json.dumps(r), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
