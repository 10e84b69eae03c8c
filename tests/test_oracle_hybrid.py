"""Pins for oracle/hybrid.py (Alg. 1 + Alg. 2; SURVEY.md §8(c.3) pins 7 and 10).

The hybrid step is an exact reformulation of full-batch training: the
pipelined, microbatched, data-parallel loss and gradients must equal the
plain sequential full-batch ones (brute force, fp64 rel <= 1e-12)."""
import numpy as np
import pytest

from oracle import hybrid, model
from synth import init_params, markov_tokens

TINY = model.GPTConfig(n_layers=2, hidden=64, heads=2, seq_len=32, vocab=256)
TINY4 = model.GPTConfig(n_layers=4, hidden=32, heads=2, seq_len=16, vocab=64)


def p64(cfg):
    p = init_params(cfg.n_layers, cfg.hidden, cfg.seq_len, cfg.vocab, seed=42, parity=True)
    return {k: v.astype(np.float64) for k, v in p.items()}


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


_REF = {}


def reference(cfg, B):
    key = (cfg, B)
    if key not in _REF:
        p = p64(cfg)
        tok = markov_tokens(B, cfg.seq_len, cfg.vocab, seed=7)
        _REF[key] = (p, tok, model.full_batch_loss_and_grads(p, cfg, tok))
    return _REF[key]


@pytest.mark.parametrize("cfg,gi", [(TINY, 1), (TINY, 2), (TINY4, 4)])
@pytest.mark.parametrize("gd", [1, 2])
@pytest.mark.parametrize("bm", [1, 2, 4])
def test_pipelined_equals_sequential(cfg, gi, gd, bm):
    B = 8
    p, tok, (loss_ref, g_ref) = reference(cfg, B)
    loss, g = hybrid.hybrid_step(p, cfg, tok, gi, gd, bm)
    assert abs(loss - loss_ref) <= 1e-12 * abs(loss_ref)
    assert set(g) == set(g_ref)
    for k in g_ref:
        assert rel(g[k], g_ref[k]) <= 1e-12, k


def test_dp_identity_and_sum():
    """Pin 10: G_data = 1 is the identity; the column sum over replicas equals
    the full-batch gradient."""
    cfg = TINY
    p, tok, (loss_ref, g_ref) = reference(cfg, 8)
    l1, g1 = hybrid.hybrid_step(p, cfg, tok, 1, 1, 8)
    for k in g_ref:
        assert np.array_equal(g1[k], g_ref[k])
    # manual replica sum
    half = [hybrid.hybrid_step(p, cfg, tok[j * 4:(j + 1) * 4], 1, 1, 4)[1] for j in range(2)]
    l2, g2 = hybrid.hybrid_step(p, cfg, tok, 1, 2, 4)
    for k in g_ref:
        # halves were normalised by M_total = 1 each; the full batch by M_total = 2
        assert rel(g2[k], (half[0][k] + half[1][k]) / 2) <= 1e-13
        assert rel(g2[k], g_ref[k]) <= 1e-12


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_schedule_timing_does_not_change_numerics(seed):
    """Random action costs reorder the schedule; accumulation order stays
    ascending per stage, so gradients are bit-identical (D-19)."""
    cfg = TINY4
    p, tok, _ = reference(cfg, 8)
    l0, g0 = hybrid.hybrid_step(p, cfg, tok, 4, 1, 1)
    l1, g1 = hybrid.hybrid_step(p, cfg, tok, 4, 1, 1, seed=seed)
    l2, g2 = hybrid.hybrid_step(p, cfg, tok, 4, 1, 1, policy="arrival", seed=seed)
    assert l0 == l1 == l2
    for k in g0:
        assert np.array_equal(g0[k], g1[k]) and np.array_equal(g0[k], g2[k])


def test_validation_errors():
    p, tok, _ = reference(TINY, 8)
    with pytest.raises(hybrid.ConfigError, match="NonDivisibleLayers"):
        hybrid.hybrid_step(p, TINY, tok, 3, 1, 1)
    with pytest.raises(hybrid.ConfigError, match="NonDivisibleBatch"):
        hybrid.hybrid_step(p, TINY, tok, 1, 3, 1)
    with pytest.raises(hybrid.ConfigError, match="NonDivisibleBatch"):
        hybrid.hybrid_step(p, TINY, tok, 1, 2, 3)


@pytest.mark.parametrize("half", ["bf16", "fp16"])
def test_half_accumulation_one_microbatch_is_rounded_exact_gradient(half):
    """grad_accum="half" (reading D-38) with one microbatch per replica: every weight matrix is
    RN(exact full-batch gradient) (a single rounding of the plain definition), every other
    tensor the exact gradient."""
    from oracle.bf16 import round_half
    cfg = TINY
    p, tok, (loss_ref, g_ref) = reference(cfg, 8)
    loss, g = hybrid.hybrid_step(p, cfg, tok, 1, 1, 8, grad_accum="half", half=half)
    assert abs(loss - loss_ref) <= 1e-12 * abs(loss_ref)
    n_half = 0
    for k in g_ref:
        if hybrid.accumulates_in_half(k):
            n_half += 1
            assert np.array_equal(g[k], round_half(g_ref[k], half).astype(np.float64)), k
        else:
            assert rel(g[k], g_ref[k]) <= 1e-12, k
    assert n_half == 4 * cfg.n_layers + 1   # w_qkv, w_o, w_fc1, w_fc2 per layer + head_w


@pytest.mark.parametrize("half,u,eta", [("bf16", 2.0 ** -8, 2.0 ** -134), ("fp16", 2.0 ** -11, 2.0 ** -25)])
@pytest.mark.parametrize("gi,gd,bm", [(1, 1, 1), (2, 1, 2), (2, 2, 1)])
def test_half_accumulation_error_bound(gi, gd, bm, half, u, eta):
    """m microbatches: each step g <- RN(g + RN(dg)) errs by at most u |dg| and u |partial sum|
    (bf16: 8 significant bits, unit roundoff u = 2^-8; fp16: 11 bits, u = 2^-11) plus, for a
    subnormal result, half the subnormal spacing eta (fp16 2^-25, bf16 2^-134), so
    |g_half - g_exact| <= sum over steps (u (|dg| + |partial|) + 2 eta) elementwise.  A dropped, doubled or sign-flipped microbatch
    breaks the bound by the size of a whole microbatch gradient."""
    cfg = TINY
    B = 8
    p, tok, (loss_ref, g_ref) = reference(cfg, B)
    _, g = hybrid.hybrid_step(p, cfg, tok, gi, gd, bm, grad_accum="half", half=half)
    m = B // (gd * bm)
    # per-step bound from the exact per-microbatch gradients of a replica's rows
    for k in g_ref:
        if not hybrid.accumulates_in_half(k):
            assert rel(g[k], g_ref[k]) <= 1e-12, k
            continue
        bound = np.zeros_like(g_ref[k])
        for j in range(gd):
            part = np.zeros_like(g_ref[k])
            for mu in range(m):
                rows = tok[(j * m + mu) * bm:(j * m + mu + 1) * bm]
                _, gm = model.full_batch_loss_and_grads(p, cfg, rows)
                dg = gm[k] * bm / B          # pre-divided by M_total (D-9)
                part = part + dg
                bound += u * (np.abs(dg) + np.abs(part)) + 2 * eta
        err = np.abs(g[k] - g_ref[k])
        assert np.all(err <= bound + 1e-30), (k, float((err - bound).max()))
        assert not np.array_equal(g[k], g_ref[k]) or m == 1


def test_half_accumulation_rejects_unknown_mode():
    with pytest.raises(hybrid.ConfigError):
        p, tok, _ = reference(TINY, 8)
        hybrid.hybrid_step(p, TINY, tok, 1, 1, 8, grad_accum="fp8")
