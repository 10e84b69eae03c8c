"""Pins for oracle/bf16.py and oracle/metrics.py (SURVEY.md §8(c.3) pins 14-16)."""
from fractions import Fraction

import numpy as np

from oracle import metrics
from oracle.bf16 import from_bf16_bits, round_bf16, round_fp16, to_bf16_bits


def test_bf16_rne_values():
    """Pin 14: 0.1 -> 0.10009765625, 1/3 -> 0.333984375 (RNE), exact values pass."""
    assert float(round_bf16(np.float32(0.1))[()]) == 0.10009765625
    assert float(round_bf16(np.float32(1 / 3))[()]) == 0.333984375
    for x in (1.0, -2.0, 0.5, 3.0, 65536.0):
        assert float(round_bf16(np.float32(x))[()]) == x
    # ties to even: 1 + 2^-8 is a tie between 1 and 1 + 2^-7 -> 1 (even mantissa)
    assert float(round_bf16(np.float32(1 + 2 ** -8))[()]) == 1.0
    assert float(round_bf16(np.float32(1 + 3 * 2 ** -8))[()]) == 1 + 2 ** -6
    assert np.isinf(round_bf16(np.float32(np.inf)))
    assert np.isnan(round_bf16(np.float32(np.nan)))


def test_bf16_vs_torch_cast():
    """Cross-check against torch's float32 -> bfloat16 cast (library routine)."""
    import torch
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(100000) * np.exp(rng.uniform(-30, 30, 100000))).astype(np.float32)
    ref = torch.tensor(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(round_bf16(x), ref)
    bits = to_bf16_bits(x)
    assert np.array_equal(from_bf16_bits(bits), ref)


def test_fp16_rne_values():
    """Pin 14 (fp16 part, N2): fp16(0.1) = 0.0999755859375; the largest finite value 65504;
    65520 (halfway to 2^16) rounds to inf; 2^-25 is a tie between 0 and the smallest
    subnormal 2^-24 -> 0 (even); 3*2^-25 -> 2^-23; ties to even at 1 + 2^-11."""
    f = lambda x: float(round_fp16(np.float32(x))[()])
    assert f(0.1) == 0.0999755859375
    assert f(65504.0) == 65504.0 and f(65519.0) == 65504.0
    assert np.isinf(f(65520.0)) and np.isinf(f(-1e6)) and f(-1e6) < 0
    assert f(2.0 ** -25) == 0.0 and f(3 * 2.0 ** -25) == 2.0 ** -23 and f(2.0 ** -24) == 2.0 ** -24
    assert f(1 + 2 ** -11) == 1.0 and f(1 + 3 * 2 ** -11) == 1 + 2 ** -9
    assert np.isnan(f(np.nan))


def test_fp16_vs_torch_cast():
    """Cross-check against torch's float32 -> float16 cast (library routine)."""
    import torch
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(100000) * np.exp(rng.uniform(-25, 15, 100000))).astype(np.float32)
    ref = torch.tensor(x).to(torch.float16).to(torch.float32).numpy()
    assert np.array_equal(round_fp16(x), ref)


def test_eq2():
    """Pin 15: Eq. 2 with t = 1, b = 2048, s = 512 -> 286102.294921875 s."""
    assert metrics.eq2_training_time(1, 2048, 512) == Fraction(286102294921875, 10**9)


def test_eq3_and_model_flops_identities():
    """Eq. 3 and model-FLOP integer forms equal their rational formulas; at
    the 12B shape the ratio Eq. 3 / model FLOPs is ~1.33 (D-25)."""
    b, s, l, h, V = 1024, 512, 48, 4512, 51200
    e3 = Fraction(96 * b * s * l * h * h) * (1 + Fraction(s, 6 * h) + Fraction(V, 16 * l * h))
    assert metrics.eq3_flops(b, s, l, h, V) == e3
    mf = Fraction(72 * b * s * l * h * h) * (1 + Fraction(s, 6 * h)) + 6 * b * s * h * V
    assert metrics.model_flops(b, s, l, h, V) == mf
    ratio = metrics.eq3_flops(b, s, l, h, V) / metrics.model_flops(b, s, l, h, V)
    assert 1.30 < ratio < 1.34
    # D2 12B-shaped 4x2, B = 1024 -> 3.831e16 model FLOPs
    assert abs(metrics.model_flops(1024, 512, 48, 4512, 51200) / 3.831e16 - 1) < 1e-3
    # D1 1.3B-shaped: 2.680e14 per 64 samples
    assert abs(metrics.model_flops(64, 512, 24, 2048, 51200) / 2.680e14 - 1) < 1e-3


def test_memory_ledger():
    """Pin 16: 20 phi = 40 GB at phi = 2e9; 4 phi + 16 bsize."""
    assert metrics.model_state_bytes(2 * 10**9) == 40 * 10**9
    assert metrics.offload_state_bytes(2 * 10**9, 16 * 10**6) == 8 * 10**9 + 256 * 10**6
    # untied 12B: 12.19e9 parameters
    assert abs(metrics.param_count(48, 4512, 512, 51200) / 12.19e9 - 1) < 1e-3
