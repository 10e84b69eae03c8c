"""world_size-2 CPU tests (gloo) of the N > 1 host plumbing: grid placement,
batch sharding (Alg. 1 l.5), unique-id broadcast, max-over-ranks timing, and
the data-parallel decomposition Alg. 1 l.13 (per-replica pre-divided
gradients SUM-all-reduced == full-batch gradient) across real processes."""
import os
import socket

import numpy as np
import pytest

from paper_2110_13005_b200 import dist as D


def test_grid_math():
    gi, gd = 4, 3   # fig:axonn-design example, 4 x 3
    seen = set()
    for r in range(gi * gd):
        i, j = D.grid_coords(r, gi)
        assert D.grid_rank(i, j, gi) == r
        seen.add((i, j))
    assert len(seen) == 12
    assert D.column_ranks(1, gi, gd) == [1, 5, 9]
    assert D.row_ranks(2, gi) == [8, 9, 10, 11]
    assert D.batch_shard(96, 3, 1) == (32, 64)
    with pytest.raises(ValueError):
        D.batch_shard(10, 3, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    from oracle import hybrid, model
    from synth import init_params, markov_tokens
    D.init_process_group(rank, world, backend="gloo")
    nid = D.share_unique_id(rank, world, lambda: bytes(range(128)))
    cfg = model.GPTConfig(n_layers=2, hidden=32, heads=2, seq_len=16, vocab=64)
    p = {k: v.astype(np.float64) for k, v in init_params(2, 32, 16, 64, seed=42).items()}
    B, bm = 8, 2
    tok = markov_tokens(B, 16, 64, seed=7)
    lo, hi = D.batch_shard(B, world, rank)
    # this replica's share, pre-divided by the microbatches of the WHOLE batch (D-9)
    m_total = B // bm
    loss = 0.0
    grads = None
    for mu in range((hi - lo) // bm):
        rows = tok[lo + mu * bm: lo + (mu + 1) * bm]
        l, c = model.stage_forward(p, cfg, 0, 1, rows[:, :-1], rows[:, 1:], m_total)
        _, g = model.stage_backward(p, cfg, 0, 1, c, 1.0)
        loss += l
        grads = g if grads is None else {k: grads[k] + g[k] for k in g}
    flat = torch.tensor(np.concatenate([grads[k].ravel() for k in sorted(grads)] + [[loss]]))
    dist.all_reduce(flat)                      # Alg. 1 l.13 SUM
    t = D.max_over_ranks(float(rank + 1), world)
    t = (t, D.gather_to_all(10.0 * rank + 0.5, world))
    q.put((rank, nid, flat.numpy(), t))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_data_parallel_gloo():
    import torch.multiprocessing as mp
    from oracle import hybrid, model
    from synth import init_params, markov_tokens
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = sorted([q.get(timeout=120) for _ in range(2)], key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert out[0][1] == out[1][1] == bytes(range(128))   # rank 0's id reached rank 1
    assert out[0][3][0] == out[1][3][0] == 2.0           # max over ranks
    assert out[0][3][1] == out[1][3][1] == [0.5, 10.5]   # gathered in rank order
    assert np.array_equal(out[0][2], out[1][2])          # both replicas hold the same sum
    cfg = model.GPTConfig(n_layers=2, hidden=32, heads=2, seq_len=16, vocab=64)
    p = {k: v.astype(np.float64) for k, v in init_params(2, 32, 16, 64, seed=42).items()}
    tok = markov_tokens(8, 16, 64, seed=7)
    loss_ref, g_ref = model.full_batch_loss_and_grads(p, cfg, tok)
    ref = np.concatenate([g_ref[k].ravel() for k in sorted(g_ref)] + [[loss_ref]])
    assert np.linalg.norm(out[0][2] - ref) <= 1e-12 * np.linalg.norm(ref)
    # and the in-process virtual-worker oracle agrees
    l2, g2 = hybrid.hybrid_step(p, cfg, tok, 1, 2, 2)
    assert abs(l2 - loss_ref) <= 1e-12 * loss_ref
