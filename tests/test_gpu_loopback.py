"""Alg. 2 on ONE GPU: the test-only loopback transport (include/axonn.h axonn_local_group).

G_inter stage contexts of one pipeline live in this process on cuda:0, each created and
driven by its own thread; messages are the production peer-copy link (copy into the
neighbour's slot mb mod pipeline_limit, then a stream-memop store of the sequence number
into its flag).  This puts the message-driven scheduler (warm-up
injection l.3-9, reaction to landed messages l.10-23, injection after stage 0's backward
l.24-26), the slot ring, the sequence numbers and backward-first dispatch (D-19) in front
of the 1-GPU driver run, against the oracle's plain full-batch result (the pipelined
reformulation is exact; oracle pin: tests/test_oracle_hybrid.py).

Cases: m > pipeline_limit (every slot reused), m < pipeline_limit (D-18), pipeline_limit 1,
G_inter 2 and 4, the 12B layer shape (h 4512: 36.96 MB messages at b_m 8, Table I/II
PAPER.md:819, 928), the offloaded optimizer over 3 steps, the fp16 build.  The stage split
cannot change a value (each stage runs the same kernels on the same bf16 inputs), so the
loopback result must also equal the single-stage run bit for bit."""
import os

import numpy as np
import pytest

from parity import assert_grads_close, oracle_mixed
from synth import init_params, markov_tokens, mixed_batch

pytestmark = pytest.mark.gpu

TINY = dict(n_layers=2, hidden=64, heads=2, seq_len=32, vocab=256)
MINI = dict(n_layers=4, hidden=256, heads=4, seq_len=128, vocab=1024)
L12B = dict(n_layers=2, hidden=4512, heads=24, seq_len=512, vocab=51200)


@pytest.fixture(autouse=True)
def _watchdog(monkeypatch):
    monkeypatch.setenv("AXONN_WATCHDOG_S", "120")   # a protocol bug fails instead of hanging


def pipeline(cfg, g_inter, mb, params, batches, steps=0, dtype="bf16", **kw):
    """Run `batches` through a loopback pipeline of g_inter stages; after each batch (when
    steps > its index) an optimizer step.  Returns (losses, grads32 of the first batch,
    final theta32, final theta16) merged over the stages."""
    from paper_2110_13005_b200.engine import (T_GRAD32, T_MASTER, T_PARAM16, AxoNN, LocalGroup,
                                              run_stages)
    grp = LocalGroup(g_inter, dtype)
    engs = run_stages(lambda i: AxoNN(g_inter, 1, mb, **cfg, rank=i, world_size=g_inter, device=0,
                                      local_group=grp, dtype=dtype, **kw), g_inter)
    try:
        for e in engs:
            e.write_all(T_MASTER, {k: params[k] for k, _, _ in e.tensors()})
        losses, g0 = [], None
        for b, tok in enumerate(batches):
            ls = run_stages(lambda i: engs[i].run_batch(tok), g_inter)
            assert len(set(ls)) == 1, ls   # C5: every stage reports the same loss
            losses.append(ls[0])
            if b == 0:
                g0 = {}
                for e in engs:
                    g0.update(e.read_all(T_GRAD32))
            if b < steps:
                run_stages(lambda i: engs[i].optimizer_step(), g_inter)
        th, t16 = {}, {}
        for e in engs:
            th.update(e.read_all(T_MASTER))
            t16.update(e.read_all(T_PARAM16))
        return losses, g0, th, t16
    finally:
        for e in engs:
            e.close()
        grp.free()


def single(cfg, mb, params, batches, steps=0, dtype="bf16", **kw):
    from paper_2110_13005_b200.engine import T_GRAD32, T_MASTER, T_PARAM16, AxoNN
    e = AxoNN(1, 1, mb, **cfg, dtype=dtype, **kw)
    try:
        e.write_all(T_MASTER, params)
        losses, g0 = [], None
        for b, tok in enumerate(batches):
            losses.append(e.run_batch(tok))
            if b == 0:
                g0 = e.read_all(T_GRAD32)
            if b < steps:
                e.optimizer_step()
        return losses, g0, e.read_all(T_MASTER), e.read_all(T_PARAM16)
    finally:
        e.close()


def bitwise_equal(a: dict, b: dict, what):
    assert set(a) == set(b), (what, set(a) ^ set(b))
    for k in a:
        assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), (what, k)


@pytest.mark.parametrize("cfg,g_inter,mb,B,limit", [
    (TINY, 2, 2, 8, 0),      # m 4 > limit 2: both slots reused twice
    (TINY, 2, 1, 8, 1),      # pipeline_limit 1: one slot, strictly alternating F / B
    (MINI, 4, 2, 16, 0),     # m 8 > limit 4
    (MINI, 4, 2, 4, 0),      # m 2 < limit 4: inject min(limit, m) (D-18)
    (MINI, 2, 4, 16, 3),     # limit 3 does not divide m 4: slot index mb mod 3 wraps unevenly
])
def test_loopback_pipeline_vs_oracle(cfg, g_inter, mb, B, limit):
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    distinct = markov_tokens(3, cfg["seq_len"], cfg["vocab"], seed=17)
    tok, counts = mixed_batch(distinct, B, seed=B + mb)
    losses, g, _, _ = pipeline(cfg, g_inter, mb, params, [tok], pipeline_limit=limit)
    loss_ref, g_ref = oracle_mixed(params, cfg, distinct, counts)
    assert abs(losses[0] - loss_ref) <= 2e-2 * abs(loss_ref), (losses[0], loss_ref)
    assert_grads_close(g, g_ref, where=f"loopback {g_inter} stages mb {mb} B {B}")
    # the stage split changes no value: bitwise equal to the single-stage run
    l1, g1, _, _ = single(cfg, mb, params, [tok])
    assert l1[0] == losses[0], (l1, losses)
    bitwise_equal(g, g1, "grad32 vs G_inter 1")


@pytest.mark.parametrize("offload", [0, 1])
def test_loopback_training_steps_equal_single_stage(offload):
    """3 x (run_batch + optimizer_step) through the loopback pipeline (offload on / off, the
    optimizer overlapping the next batch when offloaded, D-32): losses, theta32 and theta16
    bitwise equal to the single-stage run."""
    cfg = MINI
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=3)
    toks = [markov_tokens(16, cfg["seq_len"], cfg["vocab"], seed=40 + k) for k in range(3)]
    kw = dict(offload=bool(offload), bucket_elems=100_000, coarsen_k=2)
    a = pipeline(cfg, 2, 2, params, toks, steps=3, **kw)
    b = single(cfg, 2, params, toks, steps=3, **kw)
    assert a[0] == b[0], (a[0], b[0])
    bitwise_equal(a[2], b[2], "theta32")
    bitwise_equal(a[3], b[3], "theta16")


def test_loopback_fp16_pipeline_vs_oracle():
    """§8(f) N2 through the loopback: fp16 messages, static loss scale 1024, loss and every
    gradient vs the oracle at theta16 = RNE_fp16(theta) (the gradients carry S, D-11)."""
    from oracle.bf16 import round_half
    cfg = TINY
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    distinct = markov_tokens(3, cfg["seq_len"], cfg["vocab"], seed=19)
    tok, counts = mixed_batch(distinct, 8, seed=2)
    S = 1024.0
    losses, g, _, _ = pipeline(cfg, 2, 2, params, [tok], dtype="fp16", loss_scale=S)
    p16 = {k: round_half(v, "fp16") for k, v in params.items()}
    loss_ref, g_ref = oracle_mixed(p16, cfg, distinct, counts, loss_scale=S)
    assert abs(losses[0] - loss_ref / S) <= 2e-2 * abs(loss_ref / S), (losses[0], loss_ref / S)
    assert_grads_close(g, g_ref, where="loopback fp16")


def test_loopback_12b_layer_shape_vs_oracle():
    """The paper's 12B layer (h 4512, 24 heads, d 188 padded to 192, s 512, V 51200; Table I)
    at its Table II microbatch b_m 8: every message is [8, 512, 4512] bf16 = 36.96 MB.  Two
    stages of one layer each, m = 3 > pipeline_limit 2, so slot 0 is reused at full size."""
    cfg = L12B
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    distinct = markov_tokens(3, cfg["seq_len"], cfg["vocab"], seed=23)
    tok, counts = mixed_batch(distinct, 24, seed=9)
    losses, g, _, _ = pipeline(cfg, 2, 8, params, [tok])
    loss_ref, g_ref = oracle_mixed(params, cfg, distinct, counts)
    assert abs(losses[0] - loss_ref) <= 2e-2 * abs(loss_ref), (losses[0], loss_ref)
    assert_grads_close(g, g_ref, where="loopback 12B layer shape")


def test_loopback_bad_group_arguments():
    """A loopback group needs world_size == group size, and G_data > 1 needs the bf16 build
    (the fused column reduction; there is no NCCL in the loopback) (INVALID_ARG)."""
    from paper_2110_13005_b200.engine import AxoNN, AxoNNError, LocalGroup
    grp = LocalGroup(2, "fp16")
    try:
        with pytest.raises(AxoNNError) as e:
            AxoNN(1, 2, 2, **TINY, rank=0, world_size=2, device=0, local_group=grp, dtype="fp16",
                  loss_scale=1024.0)
        assert e.value.status == "INVALID_ARG"
        with pytest.raises(AxoNNError) as e:
            AxoNN(4, 1, 2, **MINI, rank=0, world_size=4, device=0, local_group=grp)
        assert e.value.status == "INVALID_ARG"
    finally:
        grp.free()


def grid_run(cfg, gi, gd, mb, params, batches, steps, **kw):
    """A G_inter x G_data grid of loopback contexts on cuda:0 (rank = j * G_inter + i): the
    pipelines of the G_data replicas plus the fused column reduction (reading D-35).  Returns
    per-rank dicts of the first batch's fp32 / half gradients (un-reduced, this replica's rows)
    and the final theta32, and the losses."""
    from paper_2110_13005_b200.engine import (T_GRAD, T_GRAD32, T_MASTER, AxoNN, LocalGroup,
                                              run_stages)
    n = gi * gd
    grp = LocalGroup(n)
    engs = run_stages(lambda r: AxoNN(gi, gd, mb, **cfg, rank=r, world_size=n, device=0,
                                      local_group=grp, **kw), n)
    try:
        for e in engs:
            e.write_all(T_MASTER, {k: params[k] for k, _, _ in e.tensors()})
        losses, g32, g16, th_pre = [], None, None, None
        for b, tok in enumerate(batches):
            ls = run_stages(lambda r: engs[r].run_batch(tok), n)
            assert len(set(ls)) == 1, ls
            losses.append(ls[0])
            if b == 0:
                g32 = [e.read_all(T_GRAD32) for e in engs]
                g16 = [e.read_all(T_GRAD) for e in engs]
                th_pre = [e.read_all(T_MASTER) for e in engs]
            if b < steps:
                run_stages(lambda r: engs[r].optimizer_step(), n)
            if b == 0:
                th_post = [e.read_all(T_MASTER) for e in engs]
        return losses, g32, g16, th_pre, th_post, [e.read_all(T_MASTER) for e in engs]
    finally:
        for e in engs:
            e.close()
        grp.free()


@pytest.mark.parametrize("cfg,gi,gd,mb,B", [(TINY, 1, 2, 2, 8), (MINI, 2, 2, 2, 16), (TINY, 1, 4, 1, 8)])
def test_loopback_fused_column_reduction_vs_oracle(cfg, gi, gd, mb, B):
    """Alg. 1 l.13 as the fused column reduction of reading D-35, on one
    GPU: G_inter x G_data contexts; replica j runs rows [j B / G_data, (j+1) B / G_data) (Alg. 1
    l.5).  Bars: the column sum of the fp32 partial gradients vs the oracle's full-batch gradient
    (cos, scale, elementwise); K9 on every replica equals the oracle's fp32 AdamW applied to the
    fp32 sum (ascending j) of the replicas' half gradients, bit for bit; all replicas end with
    identical weights."""
    from oracle import adamw
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    distinct = markov_tokens(3, cfg["seq_len"], cfg["vocab"], seed=29)
    tok, counts = mixed_batch(distinct, B, seed=B + gd)
    losses, g32, g16, th_pre, th_post, _ = grid_run(cfg, gi, gd, mb, params, [tok], steps=1,
                                                    bucket_elems=7_000, coarsen_k=2)
    loss_ref, g_ref = oracle_mixed(params, cfg, distinct, counts)
    assert abs(losses[0] - loss_ref) <= 2e-2 * abs(loss_ref), (losses[0], loss_ref)
    sc = adamw.step_scalars(1)
    for i in range(gi):
        col = [j * gi + i for j in range(gd)]
        names = list(g32[col[0]])
        gsum = {k: sum(g32[r][k].astype(np.float64) for r in col) for k in names}
        assert_grads_close(gsum, g_ref, names=names, where=f"stage {i} column sum")
        for k in names:
            g = np.zeros_like(g16[col[0]][k], dtype=np.float32)
            for r in col:   # fp32 sum in replica order of the half gradients (K9's order)
                g = (g + g16[r][k].astype(np.float32)).astype(np.float32)
            th = th_pre[col[0]][k].copy()
            m = np.zeros_like(th)
            v = np.zeros_like(th)
            adamw.adamw_step_fp32(th, m, v, g, sc)
            for r in col:
                assert np.array_equal(th_post[r][k].view(np.uint32), th.view(np.uint32)), (r, k)


def test_loopback_fused_reduction_offload_three_steps():
    """2 x 2 grid, offloaded optimizer overlapping the next batch (D-32), 3 steps: every replica
    of a stage ends with bit-identical weights, and the losses follow the single-context run
    within the bf16 tolerance (the reduction sums the replicas' half gradients in fp32, the
    single context casts one fp32 sum: not bitwise)."""
    cfg = MINI
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=3)
    toks = [markov_tokens(16, cfg["seq_len"], cfg["vocab"], seed=70 + k) for k in range(3)]
    kw = dict(offload=True, bucket_elems=100_000, coarsen_k=2)
    losses, _, _, _, _, th = grid_run(cfg, 2, 2, 2, params, toks, steps=3, **kw)
    ref = single(cfg, 2, params, toks, steps=3, **kw)
    for a, b in zip(losses, ref[0]):
        assert abs(a - b) <= 2e-2 * abs(b), (losses, ref[0])
    for i in range(2):
        for k in th[i]:
            assert np.array_equal(th[i][k].view(np.uint32), th[2 + i][k].view(np.uint32)), (i, k)


@pytest.mark.parametrize("mode", ["copy", "direct"])
def test_loopback_direct_send_equals_copy(monkeypatch, mode):
    """N3: the producing kernels store each message straight into the neighbour's slot
    (AXONN_P2P default 'direct': the top layer's output GEMM via its TMA epilogue, the stage-input
    gradient's LayerNorm backward by plain stores) or the copy engine copies it (copy).  Both
    equal the single-stage run bit for bit, with a balanced split whose top layer ends after
    its attention block (the message is x1) and with whole layers."""
    monkeypatch.setenv("AXONN_P2P", mode)
    cfg = dict(n_layers=2, hidden=64, heads=2, seq_len=32, vocab=1024)   # balanced: cut after l1's attention
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=8)
    toks = [markov_tokens(8, cfg["seq_len"], cfg["vocab"], seed=90 + k) for k in range(2)]
    for bal in (False, True):
        a = pipeline(cfg, 2, 2, params, toks, steps=2, stage_balance=bal)
        b = single(cfg, 2, params, toks, steps=2)
        assert a[0] == b[0], (bal, a[0], b[0])
        bitwise_equal(a[1], b[1], "grad32")
        bitwise_equal(a[2], b[2], "theta32")
