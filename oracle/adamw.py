"""AdamW with decoupled weight decay, monolithic and bucketed-offload forms —
oracle (test infrastructure only).

Follows:
* "run the optimizer" (Alg. 1 l.7) = Adam
  with lr 1e-3, beta 0.9/0.999 and decoupled weight decay 0.01
  (PAPER.md:841-843); eps = 1e-8 and bias correction on (reading D-13).
* Mixed precision: the optimizer converts the half-precision gradients to
  full precision, descales them by the loss scale, and updates the fp32
  master copy; theta16 is refreshed from it (D-15).  The
  paper fixes this arithmetic at single precision, so this module computes
  in numpy float32 (each elementary operation rounded once, no FMA
  contraction) in the op order of reading D-14:

      g     = g16 * inv_scale
      theta = theta * decay                      decay     = f32(1 - lr*wd)
      m     = b1 * m + omb1 * g                  omb1      = f32(1 - beta1)
      v     = b2 * v + omb2 * (g * g)            omb2      = f32(1 - beta2)
      theta = theta - step * (m / (sqrt(v) / bc2_sqrt + eps))
                                                 step      = f32(lr / (1 - beta1^t))
                                                 bc2_sqrt  = f32(sqrt(1 - beta2^t))
      theta16 = RNE_bf16(theta)

  Scalars are computed once in double and rounded once to fp32 (D-14).
* Bucketed offload: theta and s_opt live in host memory;
  buckets of ``bsize`` elements (reading D-16: elements, ascending flat
  index, ragged last bucket) are fetched into reused scratch buffers,
  updated and written back.  Adam is elementwise, so the result is
  bit-identical to the monolithic step (SPEC.md:197 idea; pin 13).

Pins: tests/test_oracle_adamw.py (closed-form step-1 values, torch AdamW
fp64 two-step values, torch fp32 within 2 ulp, g = 0 special case,
bucketed == monolithic bitwise for bsize in {1, 3, phi/2, phi}).
"""
from __future__ import annotations

import math

import numpy as np

from .bf16 import round_half


def step_scalars(t: int, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01,
                 loss_scale=1.0):
    """Host scalars for step t >= 1, computed in double and rounded once to fp32 (D-14)."""
    f = np.float32
    return dict(
        decay=f(1.0 - lr * weight_decay),
        b1=f(beta1), omb1=f(1.0 - beta1),
        b2=f(beta2), omb2=f(1.0 - beta2),
        step=f(lr / (1.0 - beta1 ** t)),
        bc2_sqrt=f(math.sqrt(1.0 - beta2 ** t)),
        eps=f(eps),
        inv_scale=f(1.0 / loss_scale),
    )


def adamw_step_fp32(theta, m, v, g16, sc: dict, half: str = "bf16"):
    """One AdamW step on float32 arrays (in place); returns theta16 (RNE to ``half``, as fp32)."""
    g = g16.astype(np.float32) * sc["inv_scale"]
    theta *= sc["decay"]
    m[...] = sc["b1"] * m + sc["omb1"] * g
    v[...] = sc["b2"] * v + sc["omb2"] * (g * g)
    denom = np.sqrt(v) / sc["bc2_sqrt"] + sc["eps"]
    theta -= sc["step"] * (m / denom)
    return round_half(theta, half)


def adamw_step_fp64(theta, m, v, g, t: int, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8,
                    weight_decay=0.01):
    """Same update in float64 with exact scalars (closed-form pins 11/12)."""
    theta = theta * (1.0 - lr * weight_decay)
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * (g * g)
    denom = np.sqrt(v) / math.sqrt(1.0 - beta2 ** t) + eps
    theta = theta - (lr / (1.0 - beta1 ** t)) * (m / denom)
    return theta, m, v


def grads_finite(g16) -> bool:
    """Overflow test of mixed precision with loss scaling (the loss is
    multiplied by a large number so small gradients survive in half precision; an overflow
    makes a gradient non-finite).  Reading D-12: when ANY gradient element of the whole
    model (every stage, after the all-reduce) is inf or NaN the optimizer step is skipped:
    theta, m, v and theta16 are left unchanged and the step counter t is not incremented."""
    return bool(np.isfinite(np.asarray(g16, dtype=np.float32)).all())


def adamw_bucketed_fp32(theta_host, m_host, v_host, g16_dev, sc: dict, bsize: int,
                        half: str = "bf16"):
    """fetch a bucket of theta and s_opt, step it on reused
    scratch buffers, offload it back.  Returns theta16 for the whole vector."""
    n = theta_host.size
    if bsize < 1:
        raise ValueError("bsize >= 1")
    cap = min(bsize, n)
    scratch_t = np.empty(cap, np.float32)          # reused device buffers
    scratch_m = np.empty(cap, np.float32)
    scratch_v = np.empty(cap, np.float32)
    theta16 = np.empty(n, np.float32)
    for lo in range(0, n, bsize):
        hi = min(lo + bsize, n)
        k = hi - lo
        t, mm, vv = scratch_t[:k], scratch_m[:k], scratch_v[:k]
        t[...] = theta_host[lo:hi]                 # H2D
        mm[...] = m_host[lo:hi]
        vv[...] = v_host[lo:hi]
        theta16[lo:hi] = adamw_step_fp32(t, mm, vv, g16_dev[lo:hi], sc, half)
        theta_host[lo:hi] = t                      # D2H
        m_host[lo:hi] = mm
        v_host[lo:hi] = vv
    return theta16
