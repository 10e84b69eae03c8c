"""Host-link roofline probe for the offloaded optimizer (A7).

One process per GPU (torchrun).  Each rank pins `--mb` MB host buffers and times
H2D alone, D2H alone and both directions at once (two streams, the offload ring's
pattern), first with rank 0 alone, then with every rank copying at the same time
(barrier-aligned).  Pinned memory is allocated either with the process's default
placement or after binding the process to the CPUs of the GPU's NUMA node (first-touch
places the pages there).  Prints one JSON line per (placement, phase, rank)."""
import argparse
import json
import os
import time

import torch
import torch.distributed as dist


def gpu_numa_node(dev: int) -> int:
    """NUMA node of the GPU's PCI function (-1 if unknown)."""
    import subprocess
    try:
        bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", str(dev)],
                             capture_output=True, text=True).stdout.strip().lower()
        dom, rest = bus.split(":", 1)
        p = f"/sys/bus/pci/devices/{dom[-4:]}:{rest}/numa_node"
        return int(open(p).read())
    except Exception:
        return -1


def node_cpus(node: int):
    p = f"/sys/devices/system/node/node{node}/cpulist"
    if not os.path.exists(p):
        return None
    cpus = set()
    for part in open(p).read().strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return cpus


def timed(fn, reps):
    """Seconds for `reps` calls (the copies run on side streams: device-synchronised wall time,
    each call moves >= 512 MB, so the launch overhead is < 0.1 %)."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=512)
    ap.add_argument("--reps", type=int, default=8)
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    node = gpu_numa_node(local)
    n = a.mb * (1 << 20)
    out = []
    all_cpus = os.sched_getaffinity(0)
    for placement in ("default", "numa_local"):
        if placement == "numa_local":
            cpus = node_cpus(node) if node >= 0 else None
            if not cpus:
                continue
            os.sched_setaffinity(0, cpus & all_cpus or cpus)
        else:
            os.sched_setaffinity(0, all_cpus)
        h_src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h_dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h_src.fill_(1)
        h_dst.fill_(2)
        d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
        d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

        def h2d():
            with torch.cuda.stream(s1):
                d_a.copy_(h_src, non_blocking=True)

        def d2h():
            with torch.cuda.stream(s2):
                h_dst.copy_(d_b, non_blocking=True)

        def duplex():
            h2d()
            d2h()

        for phase in ("alone", "all"):
            for kind, fn, mult in (("h2d", h2d, 1), ("d2h", d2h, 1), ("duplex", duplex, 2)):
                if world > 1:
                    dist.barrier()
                if phase == "alone" and rank != 0:
                    if world > 1:
                        dist.barrier()
                    continue
                fn()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                sec = timed(fn, a.reps)
                wall = time.perf_counter() - t0
                if phase == "alone" and world > 1:
                    dist.barrier()
                gbs = mult * n * a.reps / sec / 1e9
                rec = {"placement": placement, "phase": phase, "kind": kind, "rank": rank, "gpu": local,
                       "numa_node": node, "gbs": round(gbs, 2), "mb": a.mb, "reps": a.reps, "wall_s": round(wall, 3)}
                out.append(rec)
        del h_src, h_dst, d_a, d_b
    for r in out:
        print(json.dumps(r), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
