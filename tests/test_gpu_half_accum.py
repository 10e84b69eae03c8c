"""grad_accum_fp32 = 0 (reading D-38): only theta16 and the half
gradient live on the device for the weight matrices, which accumulate over the microbatches
as g <- RN(g + RN(dg_mu)); vectors and embedding tables keep fp32 accumulators.

* single context vs the oracle's half-accumulating hybrid step (oracle/hybrid.py,
  grad_accum="half"), every tensor within the parity bars (tests/parity.py);
* vectors / embeddings bit-identical to the fp32 mode (same kernels, same order), and with one
  microbatch the matrices too (RN of the same fp32 product);
* the 2 x 2 loopback grid (Alg. 2 + the fused column reduction reading every replica's half
  gradient) vs the oracle;
* the offloaded optimizer overlapping the next batch (D-32): the batch's first gradient write
  waits for the previous optimizer step, so overlap on / off end bit-identical;
* the fp16 build with a loss scale."""
import numpy as np
import pytest

from oracle import hybrid, model
from parity import assert_grads_close
from synth import init_params, markov_tokens

pytestmark = pytest.mark.gpu

TINY = dict(n_layers=2, hidden=64, heads=2, seq_len=32, vocab=256)
MINI = dict(n_layers=4, hidden=256, heads=4, seq_len=128, vocab=1024)
PAD188 = dict(n_layers=1, hidden=376, heads=2, seq_len=64, vocab=512)


@pytest.fixture(autouse=True)
def _watchdog(monkeypatch):
    monkeypatch.setenv("AXONN_WATCHDOG_S", "120")


def oracle_half(params, cfg, tok, gi, gd, mb, half="bf16", loss_scale=1.0):
    p = {k: np.asarray(v, dtype=np.float64) for k, v in params.items()}
    return hybrid.hybrid_step(p, model.GPTConfig(**cfg), tok, gi, gd, mb, loss_scale=loss_scale,
                              grad_accum="half", half=half)


def run_single(cfg, mb, params, batches, steps=0, **kw):
    from paper_2110_13005_b200.engine import T_GRAD, T_MASTER, AxoNN
    e = AxoNN(1, 1, mb, **cfg, **kw)
    try:
        e.write_all(T_MASTER, params)
        losses, g0 = [], None
        for b, tok in enumerate(batches):
            losses.append(e.run_batch(tok))
            if b == 0:
                g0 = e.read_all(T_GRAD)
            if b < steps:
                e.optimizer_step()
        return losses, g0, e.read_all(T_MASTER)
    finally:
        e.close()


@pytest.mark.parametrize("cfg,B,mb", [(TINY, 8, 2), (MINI, 16, 2), (PAD188, 8, 2), (TINY, 8, 8)])
def test_half_accum_single_vs_oracle_and_fp32_mode(cfg, B, mb):
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    tok = markov_tokens(B, cfg["seq_len"], cfg["vocab"], seed=7)
    lh, gh, _ = run_single(cfg, mb, params, [tok], grad_accum_fp32=False)
    lf, gf, _ = run_single(cfg, mb, params, [tok])
    loss_ref, g_ref = oracle_half(params, cfg, tok, 1, 1, mb)
    assert abs(lh[0] - loss_ref) <= 2e-2 * abs(loss_ref), (lh, loss_ref)
    assert lh[0] == lf[0]   # the forward does not depend on the gradient mode
    assert_grads_close(gh, g_ref, where=f"half accum {cfg} B {B} mb {mb}")
    for k in gh:
        if not hybrid.accumulates_in_half(k) or B == mb:
            assert np.array_equal(gh[k].view(np.uint32), gf[k].view(np.uint32)), k
    if B > mb:   # several microbatches: the matrices really accumulate in half
        assert any(not np.array_equal(gh[k], gf[k]) for k in gh if hybrid.accumulates_in_half(k))


def test_half_accum_grad32_of_a_matrix_is_rejected():
    from paper_2110_13005_b200.engine import T_GRAD32, AxoNN
    e = AxoNN(1, 1, 2, **TINY, grad_accum_fp32=False)
    try:
        names = [n for n, _, _ in e.tensors()]
        e.read(T_GRAD32, names.index("l0.ln1_g"))          # vectors keep fp32 accumulators
        with pytest.raises(Exception):
            e.read(T_GRAD32, names.index("l0.w_qkv"))
    finally:
        e.close()


def test_half_accum_loopback_grid_vs_oracle():
    """2 x 2 loopback grid: the column sum of the replicas' half gradients vs the oracle's,
    training 2 steps with every replica of a stage bit-identical."""
    from paper_2110_13005_b200.engine import T_GRAD, T_MASTER, AxoNN, LocalGroup, run_stages
    cfg, gi, gd, mb, B = MINI, 2, 2, 2, 16
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=5)
    toks = [markov_tokens(B, cfg["seq_len"], cfg["vocab"], seed=30 + k) for k in range(2)]
    n = gi * gd
    grp = LocalGroup(n)
    engs = run_stages(lambda r: AxoNN(gi, gd, mb, **cfg, rank=r, world_size=n, device=0,
                                      local_group=grp, grad_accum_fp32=False), n)
    try:
        for e in engs:
            e.write_all(T_MASTER, {k: params[k] for k, _, _ in e.tensors()})
        ls = run_stages(lambda r: engs[r].run_batch(toks[0]), n)
        assert len(set(ls)) == 1, ls
        g16 = [e.read_all(T_GRAD) for e in engs]
        run_stages(lambda r: engs[r].optimizer_step(), n)
        run_stages(lambda r: engs[r].run_batch(toks[1]), n)
        run_stages(lambda r: engs[r].optimizer_step(), n)
        th = [e.read_all(T_MASTER) for e in engs]
    finally:
        for e in engs:
            e.close()
        grp.free()
    loss_ref, g_ref = oracle_half(params, cfg, toks[0], gi, gd, mb)
    assert abs(ls[0] - loss_ref) <= 2e-2 * abs(loss_ref)
    g = {}
    for i in range(gi):
        for k in g16[i]:
            g[k] = g16[i][k].astype(np.float64) + g16[gi + i][k]   # replicas j = 0, 1
    assert_grads_close(g, g_ref, where="half accum 2x2")
    for i in range(gi):
        for k in th[i]:
            assert np.array_equal(th[i][k].view(np.uint32), th[gi + i][k].view(np.uint32)), (i, k)


def test_half_accum_offload_overlap_bitwise():
    """Offloaded optimizer, 3 steps: overlapping the next batch (D-32) changes nothing; the
    first half-gradient write of a batch waits for the previous optimizer step."""
    cfg = MINI
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=9)
    toks = [markov_tokens(16, cfg["seq_len"], cfg["vocab"], seed=50 + k) for k in range(3)]
    kw = dict(offload=True, bucket_elems=100_000, coarsen_k=2, grad_accum_fp32=False)
    a = run_single(cfg, 2, params, toks, steps=3, overlap_next_batch=True, **kw)
    b = run_single(cfg, 2, params, toks, steps=3, overlap_next_batch=False, **kw)
    assert a[0] == b[0]
    for k in a[2]:
        assert np.array_equal(a[2][k].view(np.uint32), b[2][k].view(np.uint32)), k


def test_half_accum_fp16_vs_oracle():
    """fp16 build, loss scale 1024: the scaled gradient accumulates in fp16 (the paper's
    format); vs the oracle with half='fp16' (gradients carry the scale S)."""
    cfg, B, mb, S = MINI, 16, 2, 1024.0
    from oracle.bf16 import round_fp16
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    p16 = {k: round_fp16(v) for k, v in params.items()}
    tok = markov_tokens(B, cfg["seq_len"], cfg["vocab"], seed=7)
    lh, gh, _ = run_single(cfg, mb, p16, [tok], dtype="fp16", loss_scale=S, grad_accum_fp32=False)
    loss_ref, g_ref = oracle_half(p16, cfg, tok, 1, 1, mb, half="fp16", loss_scale=S)
    loss_ref /= S   # the library reports the unscaled loss
    assert abs(lh[0] - loss_ref) <= 2e-2 * abs(loss_ref), (lh, loss_ref)
    assert_grads_close(gh, g_ref, where="half accum fp16")
