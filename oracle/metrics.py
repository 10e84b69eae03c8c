"""Throughput metrics and the model-state memory ledger — oracle (test
infrastructure only).

* Eq. 2: estimated training time = 3e11 * t / (b * s);
  the garbled "3e10^{11}" is read as 3x10^11 tokens (reading D-24).
* Eq. 3: flop/batch = 96 b s l h^2 (1 + s/6h + V/16lh)
  (Narayanan's count, which credits activation recompute).
* Model FLOPs (reading D-25/D-26): 72 b s l h^2 (1 + s/6h) + 6 b s h V — the
  executed forward+backward contraction FLOPs with no recompute, attention
  counted un-halved as in Eq. 3.
* Memory: 20 phi bytes of model state (4 theta + 4 grad +
  2 theta16 + 2 grad16 + 8 s_opt); with the offload optimisation
  4 phi + 16 bsize.

All in exact integer / rational arithmetic.  Pins: tests/test_oracle_misc.py
(Eq. 2 at t = 1, b = 2048, s = 512 -> 286102.294921875 s; 40 GB at
phi = 2e9; 8.256 GB at bsize = 16M; Eq. 3 / model-FLOP ratio identities).
"""
from fractions import Fraction


def model_flops(b: int, s: int, l: int, h: int, V: int) -> int:
    """72 b s l h^2 (1 + s/(6h)) + 6 b s h V, exactly (= 72bslh^2 + 12bs^2lh + 6bshV)."""
    return 72 * b * s * l * h * h + 12 * b * s * s * l * h + 6 * b * s * h * V


def eq3_flops(b: int, s: int, l: int, h: int, V: int) -> int:
    """96 b s l h^2 (1 + s/6h + V/16lh), exactly (= 96bslh^2 + 16bs^2lh + 6bshV)."""
    return 96 * b * s * l * h * h + 16 * b * s * s * l * h + 6 * b * s * h * V


def eq2_training_time(t: float, b: int, s: int) -> Fraction:
    """3e11 * t / (b s) seconds."""
    return Fraction(300_000_000_000) * Fraction(t) / (b * s)


def param_count(l: int, h: int, s: int, V: int) -> int:
    """Untied GPT (reading D-3): embeddings V h + s h, 12 h^2 + 13 h per layer, final LN 2h, head V h."""
    return V * h + s * h + l * (12 * h * h + 13 * h) + 2 * h + V * h


def model_state_bytes(phi: int) -> int:
    """20 phi."""
    return 4 * phi + 4 * phi + 2 * phi + 2 * phi + 8 * phi


def offload_state_bytes(phi: int, bsize: int) -> int:
    """4 phi + 16 bsize."""
    return 2 * phi + 2 * phi + 4 * bsize + 8 * bsize + 4 * bsize
