"""Round-to-nearest-even fp32 -> bfloat16 (value returned as float32).

Mixed precision keeps a half-precision copy theta16 of the fp32 weights
(PAPER.md:193-206); on B200 the half format is bfloat16 (reading D-31) and
theta16 = RNE(theta32) after every optimizer bucket (reading D-15).
Pinned by tests/test_oracle_misc.py (0.1 -> 0.10009765625, 1/3 ->
0.333984375, ties-to-even cases, NaN/Inf passthrough, torch cast cross-check).
"""
import numpy as np


def round_bf16(x) -> np.ndarray:
    """RNE of float32 values to bf16, returned as float32 arrays."""
    f = np.array(x, dtype=np.float32, order="C")   # keeps 0-d inputs 0-d
    bits = f.view(np.uint32).astype(np.uint64)
    # round-to-nearest-even on the low 16 bits
    lsb = (bits >> np.uint64(16)) & np.uint64(1)
    rounded = (bits + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    out = rounded.astype(np.uint32)
    nan = np.isnan(f)
    out = np.where(nan, (f.view(np.uint32) | np.uint32(0x00400000)) & np.uint32(0xFFFF0000), out)
    return out.astype(np.uint32).view(np.float32)


def to_bf16_bits(x) -> np.ndarray:
    """uint16 bit patterns of RNE(x)."""
    return (round_bf16(x).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def from_bf16_bits(b) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def round_fp16(x) -> np.ndarray:
    """RNE of float32 values to IEEE binary16 (the paper's V100 half format,
    PAPER.md:202-206; reading D-31 variant N2), returned as float32.  Overflow
    beyond 65504 (after rounding) gives +-inf, tiny values become subnormal.
    Pinned by tests/test_oracle_misc.py (0.1 -> 0.0999755859375, 65520 -> inf,
    2^-25 ties to 0, torch cast cross-check)."""
    with np.errstate(over="ignore"):   # overflow to +-inf is the defined result
        return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float32)


def round_half(x, half: str = "bf16") -> np.ndarray:
    """RNE to the 16-bit format of theta16 / the gradients: 'bf16' or 'fp16'."""
    if half == "bf16":
        return round_bf16(x)
    if half == "fp16":
        return round_fp16(x)
    raise ValueError(half)
