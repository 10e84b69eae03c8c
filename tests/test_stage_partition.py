"""The stage split of stage_balance (readings D-21b / D-21c in DESIGN.md): host logic behind
axonn_stage_partition, callable without a GPU.

Pinned against brute force: on small models every split of the 2l residual blocks into
G_inter contiguous non-empty ranges is enumerated, and the library's choice must reach the
minimum over all of them of the largest stage cost (forward FLOPs per token: attention block
8h^2 + 4 * 2sh, MLP block 16h^2, LM head 2hV on the last stage), each divided by its stage's
speed.  Speeds only rescale costs, so uniform speeds equal NULL and a slower stage never gains
blocks."""
import ctypes as C
import itertools
import math

import pytest

from paper_2110_13005_b200 import _lib

W_ATT = 4.0   # attention-core weight of the cost model (reading D-21b)


def partition(n_layers, hidden, seq, vocab, P, speed=None):
    lib = _lib.load("bf16")
    mc = _lib.ModelCfg(n_layers, hidden, 2, seq, vocab, 42, 0)
    sp = None if speed is None else (C.c_double * P)(*speed)
    out = (C.c_int * (P + 1))()
    rc = lib.axonn_stage_partition(C.byref(mc), P, sp, out)
    return rc, list(out)


def stage_costs(bounds, n_layers, h, s, V, speed):
    P = len(bounds) - 1
    blk = [(16 * h * h) if k & 1 else (8 * h * h + W_ATT * 2 * s * h) for k in range(2 * n_layers)]
    return [(sum(blk[bounds[i]:bounds[i + 1]]) + (2 * h * V if i == P - 1 else 0)) / speed[i]
            for i in range(P)]


def brute_min(n_layers, h, s, V, P, speed):
    nb = 2 * n_layers
    best = math.inf
    for cuts in itertools.combinations(range(1, nb), P - 1):
        b = [0, *cuts, nb]
        best = min(best, max(stage_costs(b, n_layers, h, s, V, speed)))
    return best


CASES = [  # (n_layers, hidden, seq, vocab, P, speed)
    (4, 64, 32, 256, 2, None),
    (4, 64, 32, 4096, 2, None),          # heavy head: the last stage sheds blocks
    (6, 128, 64, 1024, 3, None),
    (6, 128, 64, 1024, 3, [1.0, 0.8, 1.0]),
    (5, 96, 32, 2048, 4, [1.0, 1.0, 0.9, 1.0]),
    (8, 64, 512, 8192, 4, [0.95, 1.0, 1.05, 0.9]),
    (3, 64, 32, 256, 6, None),           # 2l == G_inter: one block per stage
]


@pytest.mark.parametrize("case", CASES)
def test_partition_reaches_brute_force_minimum(case):
    L, h, s, V, P, speed = case
    rc, b = partition(L, h, s, V, P, speed)
    assert rc == 0
    assert b[0] == 0 and b[-1] == 2 * L and all(b[i] < b[i + 1] for i in range(P))
    sp = speed or [1.0] * P
    got = max(stage_costs(b, L, h, s, V, sp))
    assert got <= brute_min(L, h, s, V, P, sp) * (1 + 1e-9)


def test_uniform_speed_equals_null_and_scale_invariant():
    for L, h, s, V, P, _ in CASES:
        _, b0 = partition(L, h, s, V, P)
        assert partition(L, h, s, V, P, [1.0] * P)[1] == b0
        assert partition(L, h, s, V, P, [1413.7] * P)[1] == b0


def test_slower_stage_gets_no_more_blocks():
    """The 24B 4x1 shape (48 blocks over 4 stages): slowing stage 2 by 10 % moves at least one
    block off it and never adds one."""
    L, h, s, V, P = 24, 6336, 512, 51200, 4
    _, b0 = partition(L, h, s, V, P)
    _, b1 = partition(L, h, s, V, P, [1.0, 1.0, 0.9, 1.0])
    n0 = [b0[i + 1] - b0[i] for i in range(P)]
    n1 = [b1[i + 1] - b1[i] for i in range(P)]
    assert n1[2] < n0[2]
    for slow in range(P):
        sp = [1.0] * P
        sp[slow] = 0.8
        _, b = partition(L, h, s, V, P, sp)
        assert b[slow + 1] - b[slow] <= n0[slow]


@pytest.mark.parametrize("bad", [[1.0, 0.0], [1.0, -1.0], [1.0, float("nan")], [1.0, float("inf")]])
def test_bad_speed_rejected(bad):
    rc, _ = partition(4, 64, 32, 256, 2, bad)
    assert rc == -1   # AXONN_ERR_INVALID_ARG


def test_init_rejects_bad_speed_before_device():
    from paper_2110_13005_b200.engine import AxoNN, AxoNNError
    with pytest.raises(AxoNNError) as e:
        AxoNN(2, 1, 1, n_layers=2, hidden=64, heads=2, seq_len=32, vocab=256, world_size=2,
              nccl_id=b"x" * 128, stage_balance=True, stage_speed=[1.0, 0.0])
    assert e.value.status == "INVALID_ARG"


def test_calibrate_speed_validates_and_needs_gpu():
    lib = _lib.load("bf16")
    tf = C.c_double(-1.0)
    assert lib.axonn_calibrate_speed(0, 100, 256, 256, 4, C.byref(tf)) == -1   # M < 128
    assert lib.axonn_calibrate_speed(0, 256, 256, 256, 0, C.byref(tf)) == -1   # iters < 1
    assert lib.axonn_calibrate_speed(0, 256, 256, 256, 100001, C.byref(tf)) == -1
    import torch
    if not torch.cuda.is_available():
        assert lib.axonn_calibrate_speed(0, 256, 256, 256, 4, C.byref(tf)) == -6   # AXONN_ERR_CUDA
