"""Shared GPU-vs-oracle comparison helpers of the parity tests (test infrastructure).

Bars (BASELINE.json north_star, written out per tensor):
* cosine(g, g_ref) >= 0.999 (north_star);
* scale: | ||g|| / ||g_ref|| - 1 | <= 1e-2 -- cosine is blind to a constant factor (a gradient
  pre-divided by the wrong microbatch count, a missing loss-scale descale, a doubled sum), and
  AdamW is nearly scale-invariant, so a loss-trajectory test would not see one either;
* elementwise: max |g - g_ref| <= 0.05 max |g_ref| -- a few wrong rows (e.g. of tok_emb, where
  one microbatch's tokens touch ~0.1 % of the rows) can hide inside 0.1 % of cosine.
Derivation of the two new bounds: bf16 operands carry a relative rounding error of 2^-9 per
element; the fp32-accumulated products and sums over K terms keep the error of a gradient
entry near 2^-9 of the magnitude of its largest contributing terms, i.e. well under 1 % of
max |g_ref| and of the norm, so 1e-2 and 5e-2 leave margin without admitting a structural
error (a wrong row is O(100 %) of its entries, a wrong scale >= 2x)."""
from __future__ import annotations

import numpy as np


def cos(a, b) -> float:
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    if na < 1e-30 and nb < 1e-30:
        return 1.0
    return float((a * b).sum() / (na * nb))


def grad_errors(g: np.ndarray, ref: np.ndarray):
    """(cosine, norm ratio - 1, max|g - ref| / max|ref|) of one tensor."""
    a = np.asarray(g, dtype=np.float64).ravel()
    r = np.asarray(ref, dtype=np.float64).ravel()
    na, nr = np.linalg.norm(a), np.linalg.norm(r)
    if na < 1e-30 and nr < 1e-30:
        return 1.0, 0.0, 0.0
    inf_r = np.abs(r).max()
    return cos(a, r), (na / nr - 1.0) if nr > 0 else np.inf, float(np.abs(a - r).max() / inf_r) if inf_r > 0 else np.inf


def assert_grads_close(g: dict, g_ref: dict, cos_min=0.999, norm_tol=1e-2, inf_tol=5e-2, names=None,
                       where=""):
    """Every tensor of g_ref (or of ``names``) present in g and within the three bars."""
    keys = list(g_ref) if names is None else list(names)
    bad = []
    for k in keys:
        assert k in g, (where, "missing", k)
        c, nr, inf = grad_errors(g[k], g_ref[k])
        if not (c >= cos_min and abs(nr) <= norm_tol and inf <= inf_tol):
            bad.append((k, round(c, 6), round(nr, 5), round(inf, 4)))
    assert not bad, (where, "cos / norm-1 / inf", bad[:8])


def oracle_mixed(params: dict, cfg: dict, distinct: np.ndarray, counts: np.ndarray, loss_scale=1.0):
    """Exact loss and gradient of a synth.mixed_batch batch from its distinct sequences:
    the batch-mean loss and its gradient are the count-weighted means of the per-sequence
    ones (every row of a causal LM batch is independent; D-9)."""
    from oracle import model
    p64 = {k: np.asarray(v, dtype=np.float64) for k, v in params.items()}
    c = model.GPTConfig(**cfg)
    B = int(counts.sum())
    loss, grads = 0.0, None
    for i, n in enumerate(counts):
        if n == 0:
            continue
        li, gi = model.full_batch_loss_and_grads(p64, c, distinct[i:i + 1], loss_scale)
        loss += n * li / B
        if grads is None:
            grads = {k: v * (n / B) for k, v in gi.items()}
        else:
            for k, v in gi.items():
                grads[k] += v * (n / B)
    return loss, grads
