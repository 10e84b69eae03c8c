"""Process-group bootstrap (PyTorch is plumbing only).

One process per GPU.  torch.distributed (gloo, over
127.0.0.1 rendezvous) is used to broadcast rank 0's 128-byte ncclUniqueId and
for host-side barriers / max-over-ranks timing; every data-path collective
(P2P activations/gradients, gradient all-reduce) is issued by libaxonn on its
own NCCL communicators.

Grid placement (reading D-29): world_rank = j * G_inter + i, i = stage
(position in the row = pipeline), j = replica (column = data-parallel group),
PAPER.md:294-300."""
from __future__ import annotations

import os


def grid_coords(rank: int, g_inter: int) -> tuple[int, int]:
    """(stage i, replica j) of a world rank."""
    return rank % g_inter, rank // g_inter


def grid_rank(stage: int, replica: int, g_inter: int) -> int:
    return replica * g_inter + stage


def column_ranks(stage: int, g_inter: int, g_data: int) -> list[int]:
    """The data-parallel group of stage i (a column of the grid, Alg. 1 l.13)."""
    return [grid_rank(stage, j, g_inter) for j in range(g_data)]


def row_ranks(replica: int, g_inter: int) -> list[int]:
    """The pipeline of replica j (a row of the grid, Alg. 2)."""
    return [grid_rank(i, replica, g_inter) for i in range(g_inter)]


def batch_shard(batch: int, g_data: int, replica: int) -> tuple[int, int]:
    """Rows [lo, hi) of the batch consumed by replica j (Alg. 1 l.5)."""
    if batch % g_data:
        raise ValueError("NonDivisibleBatch")
    per = batch // g_data
    return replica * per, (replica + 1) * per


def env_rank_world() -> tuple[int, int, int]:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def init_process_group(rank: int, world: int, backend: str = "gloo"):
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return dist


def share_unique_id(rank: int, world: int, make_id) -> bytes:
    """Rank 0 calls ``make_id()`` (-> 128 bytes); every rank returns it."""
    if world == 1:
        return b"\0" * 128
    import torch.distributed as dist
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def nccl_unique_id() -> bytes:
    import ctypes as C

    from . import _lib
    buf = C.create_string_buffer(128)
    rc = _lib.load().axonn_get_unique_id(buf)
    if rc != 0:
        raise RuntimeError(f"axonn_get_unique_id failed: {rc}")
    return buf.raw


def max_over_ranks(value: float, world: int) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_all(value: float, world: int) -> list[float]:
    """Every rank's value, in rank order (gloo all_gather)."""
    if world == 1:
        return [value]
    import torch
    import torch.distributed as dist
    out = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(out, torch.tensor([value], dtype=torch.float64))
    return [float(t.item()) for t in out]


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
