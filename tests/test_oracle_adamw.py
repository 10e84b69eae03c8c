"""Pins for oracle/adamw.py (SURVEY.md §8(c.3) pins 11-13)."""
import math

import numpy as np
import pytest

from oracle import adamw
from oracle.bf16 import round_bf16
from synth import adam_test_state


def test_step1_closed_form_fp64():
    """Pin 11: step 1 gives theta1 = theta0 (1 - lr wd) - lr g / (|g| + eps)
    (bias corrections cancel: m_hat = g, v_hat = g^2)."""
    lr, wd, eps = 1e-3, 0.01, 1e-8
    for th0, g, expect in [(1.0, 1.0, 0.99899000001), (-0.5, 2e-3, -0.500994995000025),
                           (0.02, -3e-5, 0.020999466777740755)]:
        th, m, v = adamw.adamw_step_fp64(np.array([th0]), np.zeros(1), np.zeros(1),
                                         np.array([g]), 1)
        closed = th0 * (1 - lr * wd) - lr * g / (abs(g) + eps)
        assert th[0] == pytest.approx(closed, rel=1e-15)
        assert th[0] == pytest.approx(expect, rel=1e-14)
    th, m, v = adamw.adamw_step_fp64(np.array([0.7]), np.zeros(1), np.zeros(1), np.zeros(1), 1)
    assert m[0] == 0 and v[0] == 0 and th[0] == 0.7 * (1 - lr * wd)


def test_two_steps_vs_torch_fp64():
    """Pin 12: two steps vs torch.optim.AdamW(foreach=False) in fp64."""
    import torch
    th0 = np.array([1.0, -0.5, 0.02, 0.0])
    gs = [np.array([1.0, 2e-3, -3e-5, 0.0]), np.array([0.5, -1e-3, 4e-5, 1e-6])]
    th, m, v = th0.copy(), np.zeros(4), np.zeros(4)
    for t, g in enumerate(gs, start=1):
        th, m, v = adamw.adamw_step_fp64(th, m, v, g, t)
    expect = np.array([0.9980478304829816, -0.5012563204050299, 0.020805801087638385,
                       -0.000733762450049168])
    np.testing.assert_allclose(th, expect, rtol=1e-15, atol=0)
    p = torch.nn.Parameter(torch.tensor(th0, dtype=torch.float64))
    opt = torch.optim.AdamW([p], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01,
                            foreach=False)
    for g in gs:
        p.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
    np.testing.assert_allclose(th, p.detach().numpy(), rtol=1e-15, atol=1e-19)


def test_fp32_vs_torch_fp32_within_4ulp():
    """The fp32 D-14 op order agrees with torch's fp32 AdamW to <= 4 ulp of the operands
    (torch uses lerp for m; same maths, different rounding path)."""
    import torch
    n = 4096
    theta, m, v, g = adam_test_state(n, seed=3)
    m[:] = 0
    v[:] = 0
    th = theta.copy()
    p = torch.nn.Parameter(torch.tensor(theta))
    opt = torch.optim.AdamW([p], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01,
                            foreach=False)
    mm, vv = m.copy(), v.copy()
    for t in (1, 2, 3):
        gt = (g * t).astype(np.float32)
        adamw.adamw_step_fp32(th, mm, vv, gt, adamw.step_scalars(t))
        p.grad = torch.tensor(gt)
        opt.step()
    ref = p.detach().numpy()
    # ulps of the operands of the final subtraction (the result can cancel)
    scale = np.maximum(np.abs(theta), np.abs(ref)).astype(np.float32)
    assert np.all(np.abs(th - ref) <= 4 * np.spacing(scale))


def test_fp32_matches_fp64_closely():
    n = 1 << 14
    theta, m, v, g = adam_test_state(n, seed=5)
    sc = adamw.step_scalars(7)
    th32, m32, v32 = theta.copy(), m.copy(), v.copy()
    adamw.adamw_step_fp32(th32, m32, v32, g, sc)
    th64, m64, v64 = adamw.adamw_step_fp64(theta.astype(np.float64), m.astype(np.float64),
                                           v.astype(np.float64), g.astype(np.float64), 7)
    assert np.linalg.norm(th32 - th64) / np.linalg.norm(th64) < 1e-6
    assert np.linalg.norm(m32 - m64) / np.linalg.norm(m64) < 1e-6
    assert np.linalg.norm(v32 - v64) / np.linalg.norm(v64) < 1e-6


@pytest.mark.parametrize("bsize", [1, 3, 500, 1000, 10**7])
def test_bucketed_equals_monolithic_bitwise(bsize):
    """Pin 13: bucketed offload == monolithic bitwise, bsize in {1, 3, phi/2, phi, > phi}."""
    n = 1000
    theta, m, v, g = adam_test_state(n, seed=8)
    sc = adamw.step_scalars(3)
    a = [theta.copy(), m.copy(), v.copy()]
    t16a = adamw.adamw_step_fp32(*a, g, sc)
    b = [theta.copy(), m.copy(), v.copy()]
    t16b = adamw.adamw_bucketed_fp32(*b, g, sc, bsize)
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    assert np.array_equal(t16a.view(np.uint32), t16b.view(np.uint32))
    assert np.array_equal(t16a, round_bf16(a[0]))


def test_step_scalars_rounded_once():
    sc = adamw.step_scalars(1)
    assert sc["step"] == np.float32(1e-3 / (1 - 0.9))
    assert sc["bc2_sqrt"] == np.float32(math.sqrt(1 - 0.999))
    assert sc["decay"] == np.float32(1 - 1e-5)


def test_overflow_skip_rule():
    """Reading D-12 (PAPER.md:198-201 loss scaling; SPEC.md:181 NonFiniteGradient): one inf or
    NaN anywhere skips the step; finite gradients of any magnitude do not."""
    g = np.zeros(1000, np.float32)
    assert adamw.grads_finite(g)
    g[17] = 65504.0
    assert adamw.grads_finite(g)
    for bad in (np.inf, -np.inf, np.nan):
        h = g.copy()
        h[999] = bad
        assert not adamw.grads_finite(h)
    # fp16 overflow of a sum of two finite values (what the column all-reduce can produce)
    from oracle.bf16 import round_fp16
    assert not adamw.grads_finite(round_fp16(np.float32(60000.0) + np.float32(60000.0)))


def test_fp16_theta16_is_rne_fp16():
    """N2: with half='fp16' theta16 = RNE_fp16(theta32), and theta32/m/v
    are bit-identical to the bf16 run (the half format only changes theta16)."""
    from oracle.bf16 import round_fp16
    rng = np.random.default_rng(3)
    th = (rng.standard_normal(4096) * 0.02).astype(np.float32)
    m = (rng.standard_normal(4096) * 1e-3).astype(np.float32)
    v = np.abs(rng.standard_normal(4096) * 1e-6).astype(np.float32)
    g = round_fp16((rng.standard_normal(4096) * 1e-3).astype(np.float32))
    sc = adamw.step_scalars(3, loss_scale=1024.0)
    a = [th.copy(), m.copy(), v.copy()]
    b = [th.copy(), m.copy(), v.copy()]
    t16a = adamw.adamw_step_fp32(*a, g * 1024, sc, "fp16")
    t16b = adamw.adamw_step_fp32(*b, g * 1024, sc, "bf16")
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    assert np.array_equal(t16a, round_fp16(a[0]))
    assert not np.array_equal(t16a, t16b)
