"""fp16 path (§8(f) N2): the libaxonn_fp16.so build of every kernel, with a static loss scale
S (reading D-11) and the overflow skip of reading D-12, vs the oracle.

The oracle does not emulate fp16 arithmetic (§8(c)): it evaluates the model in fp64 at
theta16 = RNE_fp16(theta32) (forward/backward use the half copy) and runs
the fp32 AdamW on the GPU's own fp16 gradients (descaled by 1/S inside the step, D-14).
Bars as for bf16 (BASELINE.json north_star): loss rel <= 2e-2, per-tensor gradient cosine
>= 0.999, AdamW bit-identical, theta16 == RNE_fp16(theta32) bitwise."""
import numpy as np
import pytest

from oracle import adamw, model
from oracle.bf16 import round_fp16
from synth import init_params, markov_tokens

pytestmark = pytest.mark.gpu

TINY = dict(n_layers=2, hidden=64, heads=2, seq_len=32, vocab=256)
MINI = dict(n_layers=4, hidden=256, heads=4, seq_len=128, vocab=1024)
PAD188 = dict(n_layers=1, hidden=376, heads=2, seq_len=64, vocab=512)
S = 1024.0


def make(cfg, mb=2, **kw):
    from paper_2110_13005_b200.engine import AxoNN
    kw.setdefault("loss_scale", S)
    return AxoNN(1, 1, mb, **cfg, dtype="fp16", **kw)


def cos(a, b):
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    if na < 1e-30 and nb < 1e-30:
        return 1.0
    return float((a * b).sum() / (na * nb))


def oracle_at_theta16(params32, cfg, tokens):
    p = {k: round_fp16(v).astype(np.float64) for k, v in params32.items()}
    return model.full_batch_loss_and_grads(p, model.GPTConfig(**cfg), tokens)


def test_library_is_fp16_and_bf16_ctx_rejected():
    from paper_2110_13005_b200 import _lib
    assert _lib.load("fp16").axonn_half_dtype() == 1
    assert _lib.load("bf16").axonn_half_dtype() == 0
    mc = _lib.ModelCfg(2, 64, 2, 32, 256, 42, 0)   # asks for bf16 from the fp16 build
    oc = _lib.OptCfg(1e-3, 0.9, 0.999, 1e-8, 0.01, 1.0, 0, 4000000, 4, 0, 0, 0)
    import ctypes as C
    ctx = C.c_void_p()
    rc = _lib.load("fp16").axonn_init(1, 1, 2, C.byref(mc), C.byref(oc), None, C.byref(ctx))
    assert rc == -1 and not ctx.value


@pytest.mark.parametrize("cfg,B,mb", [(TINY, 8, 2), (MINI, 16, 2), (PAD188, 4, 2)])
def test_fp16_step_loss_and_grads_vs_oracle(cfg, B, mb):
    from paper_2110_13005_b200.engine import T_GRAD32, T_MASTER, T_PARAM16
    eng = make(cfg, mb=mb)
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    eng.write_all(T_MASTER, params)
    p16 = eng.read_all(T_PARAM16)
    for k in params:   # theta16 = RNE_fp16(theta32) on write
        assert np.array_equal(p16[k].view(np.uint32), round_fp16(params[k]).view(np.uint32)), k
    tok = markov_tokens(B, cfg["seq_len"], cfg["vocab"], seed=7)
    loss = eng.run_batch(tok)   # unscaled (the library divides S out)
    loss_ref, g_ref = oracle_at_theta16(params, cfg, tok)
    assert abs(loss - loss_ref) <= 2e-2 * abs(loss_ref), (loss, loss_ref)
    g = eng.read_all(T_GRAD32)   # S x gradient
    worst = min((cos(g[k].astype(np.float64), g_ref[k]), k) for k in g_ref)
    assert worst[0] >= 0.999, worst
    # the scale is really applied: |g32| ~ S |g_ref|
    k = "head_w"
    ratio = np.linalg.norm(g[k]) / np.linalg.norm(g_ref[k])
    assert abs(ratio / S - 1) < 2e-2, ratio
    eng.close()


@pytest.mark.parametrize("offload", [0, 1])
def test_fp16_optimizer_bit_exact(offload):
    """AdamW on the fp16 gradients x S: theta32, m, v bit-identical to the oracle's fp32 step
    with inv_scale = 1/S, theta16 == RNE_fp16(theta32)."""
    from paper_2110_13005_b200.engine import T_ADAM_M, T_ADAM_V, T_GRAD, T_MASTER, T_PARAM16
    cfg = TINY
    eng = make(cfg, offload=bool(offload), bucket_elems=1000, coarsen_k=2)
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    eng.write_all(T_MASTER, params)
    tok = markov_tokens(8, cfg["seq_len"], cfg["vocab"], seed=7)
    for step in (1, 2):
        eng.run_batch(tok)
        g16 = eng.read_all(T_GRAD)
        for k in g16:
            assert np.array_equal(g16[k], round_fp16(g16[k])), k   # fp16 values
        th, m, v = eng.read_all(T_MASTER), eng.read_all(T_ADAM_M), eng.read_all(T_ADAM_V)
        eng.optimizer_step()
        sc = adamw.step_scalars(step, loss_scale=S)
        after, p16 = eng.read_all(T_MASTER), eng.read_all(T_PARAM16)
        for k in th:
            t_r, m_r, v_r = th[k].copy(), m[k].copy(), v[k].copy()
            t16 = adamw.adamw_step_fp32(t_r, m_r, v_r, g16[k], sc, half="fp16")
            assert np.array_equal(after[k].view(np.uint32), t_r.view(np.uint32)), (step, k)
            assert np.array_equal(p16[k].view(np.uint32), t16.view(np.uint32)), (step, k)
    eng.close()


def test_fp16_three_step_training_vs_oracle():
    from paper_2110_13005_b200.engine import T_MASTER
    cfg = TINY
    eng = make(cfg)
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    eng.write_all(T_MASTER, params)
    toks = [markov_tokens(8, cfg["seq_len"], cfg["vocab"], seed=100 + i) for i in range(3)]
    theta = {k: v.copy() for k, v in params.items()}
    mm = {k: np.zeros_like(v) for k, v in params.items()}
    vv = {k: np.zeros_like(v) for k, v in params.items()}
    for step, tok in enumerate(toks, start=1):
        loss = eng.run_batch(tok)
        eng.optimizer_step()
        loss_ref, g = oracle_at_theta16(theta, cfg, tok)
        sc = adamw.step_scalars(step, loss_scale=S)
        for k in theta:
            adamw.adamw_step_fp32(theta[k], mm[k], vv[k], round_fp16((g[k] * S).astype(np.float32)),
                                  sc, half="fp16")
        assert abs(loss - loss_ref) <= 2e-2 * abs(loss_ref), (step, loss, loss_ref)
    eng.close()


@pytest.mark.parametrize("offload", [0, 1])
def test_fp16_overflow_skips_step(offload):
    """Reading D-12: a loss scale so large that the scaled gradients overflow fp16 makes
    optimizer_step return NONFINITE with theta32 / m / v / theta16 untouched and t not
    incremented; the context stays usable (the next step's bias correction is t = 1's)."""
    from paper_2110_13005_b200.engine import (T_ADAM_M, T_ADAM_V, T_GRAD, T_MASTER, T_PARAM16,
                                              AxoNNError)
    cfg = TINY
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    tok = markov_tokens(8, cfg["seq_len"], cfg["vocab"], seed=7)
    eng = make(cfg, loss_scale=2.0 ** 40, offload=bool(offload), bucket_elems=1000)
    eng.write_all(T_MASTER, params)
    before = [eng.read_all(w) for w in (T_MASTER, T_ADAM_M, T_ADAM_V, T_PARAM16)]
    eng.run_batch(tok)
    g16 = eng.read_all(T_GRAD)
    assert not adamw.grads_finite(np.concatenate([v.reshape(-1) for v in g16.values()]))
    with pytest.raises(AxoNNError) as e:
        eng.optimizer_step()
    assert e.value.status == "NONFINITE"
    after = [eng.read_all(w) for w in (T_MASTER, T_ADAM_M, T_ADAM_V, T_PARAM16)]
    for a, b in zip(before, after):
        for k in a:
            assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), k
    eng.close()
    # a finite step after a skip: inject one inf through the GRAD write path, then redo
    eng = make(cfg, offload=bool(offload), bucket_elems=1000)
    eng.write_all(T_MASTER, params)
    eng.run_batch(tok)
    g = eng.read(T_GRAD, 3)
    g.reshape(-1)[5] = np.nan
    eng.write(T_GRAD, 3, g)
    with pytest.raises(AxoNNError):
        eng.optimizer_step()
    eng.run_batch(tok)
    g16 = eng.read_all(T_GRAD)
    th, m, v = eng.read_all(T_MASTER), eng.read_all(T_ADAM_M), eng.read_all(T_ADAM_V)
    eng.optimizer_step()
    sc = adamw.step_scalars(1, loss_scale=S)   # t = 1: the skipped step did not count
    after = eng.read_all(T_MASTER)
    for k in th:
        t_r = th[k].copy()
        adamw.adamw_step_fp32(t_r, m[k].copy(), v[k].copy(), g16[k], sc, half="fp16")
        assert np.array_equal(after[k].view(np.uint32), t_r.view(np.uint32)), k
    eng.close()
