"""Alg. 1 hybrid inter-layer x data-parallel step over G_inter x G_data
virtual workers — oracle (test infrastructure only).

* Grid g^{i,j}: i = stage (row position), j = replica (PAPER.md:294-300,
  reading D-29).
* Alg. 1 l.4-5: replica j takes rows [j*B/G_data, (j+1)*B/G_data) of the
  batch.
* Alg. 1 l.11-12 / Alg. 2: inter-layer step of each row, driven by the
  schedule simulator, with stage forward/backward payloads from ``model``.
  Microbatch mu of replica j is rows [mu*b_m, (mu+1)*b_m) of its shard
  (Alg. 2 l.2).
* Loss pre-divided by M_total = B / b_m, the number of microbatches in the
  whole batch (D-9).
* Alg. 1 l.13: SUM all-reduce of each stage's gradients over its column
  (D-10), replicas summed in ascending j.
* Weight gradients accumulate over microbatches in execution order, which
  the schedule guarantees is ascending microbatch id (D-19; asserted here).
* grad_accum="half" (reading D-38, the memory optimisation of PAPER.md:675-680:
  "only the half precision model parameters (theta16) and gradients
  (grad theta16) reside on the GPU ... grad theta deleted"): the weight
  matrices (``HALF_ACCUM``) accumulate in the half format, per microbatch
  g <- RN(g + RN(dg_mu)); every other tensor accumulates exactly (as with
  "fp32") and is rounded once by the caller's comparison.  The column SUM
  then adds the replicas' half gradients.  Pinned by tests/test_oracle_hybrid.py
  (one microbatch: RN of the exact gradient; bf16-exact increments: equal to
  the exact sum; the deviation from the exact sum within m half-ulps).

Pinned by tests/test_oracle_hybrid.py: equals ``model.full_batch_loss_and_grads``
(the plain definition) to fp64 rounding for every valid
(G_inter, G_data, b_m) in {1,2,4} x {1,2} x {1,2,4} on the tiny config.
"""
from __future__ import annotations

import numpy as np

from . import model, schedule
from .bf16 import round_half

# leaf names of the tensors that accumulate in the half format under grad_accum="half" (D-38)
HALF_ACCUM = ("w_qkv", "w_o", "w_fc1", "w_fc2", "head_w")


def accumulates_in_half(name: str) -> bool:
    return name.split(".")[-1] in HALF_ACCUM


class ConfigError(ValueError):
    """SPEC.md:40-48 style validation errors."""


def validate(cfg: model.GPTConfig, g_inter: int, g_data: int, microbatch: int, batch: int):
    if g_inter < 1 or g_data < 1 or microbatch < 1:
        raise ConfigError("InvalidArg")
    if cfg.n_layers % g_inter:
        raise ConfigError("NonDivisibleLayers")
    if cfg.hidden % cfg.heads:
        raise ConfigError("InvalidArg: hidden % heads")
    if batch % (g_data * microbatch):
        raise ConfigError("NonDivisibleBatch")


def split_stage_params(params: dict, cfg: model.GPTConfig, g_inter: int):
    """nn_shard for each stage i (Alg. 1 l.2)."""
    return [{n: params[n] for n in model.stage_param_names(cfg, i, g_inter)}
            for i in range(g_inter)]


def hybrid_step(params: dict, cfg: model.GPTConfig, tokens, g_inter: int, g_data: int,
                microbatch: int, loss_scale: float = 1.0, policy: str = "backward_first",
                seed: int | None = None, grad_accum: str = "fp32", half: str = "bf16"):
    """One data_parallel_step (Alg. 1 l.11-14) on every g^{i,j}.

    Returns (loss, grads) where loss = sum over all microbatches of the
    pre-divided loss (= S * batch-mean CE) and grads maps every parameter
    name to its column-summed gradient (what every replica holds after the
    all-reduce)."""
    if grad_accum not in ("fp32", "half"):
        raise ConfigError("InvalidArg: grad_accum")
    tokens = np.asarray(tokens)
    B = tokens.shape[0]
    validate(cfg, g_inter, g_data, microbatch, B)
    shard = B // g_data
    m = shard // microbatch
    m_total = B // microbatch
    shards = split_stage_params(params, cfg, g_inter)
    per_replica = []
    loss_total = 0.0
    for j in range(g_data):                                   # rows of the grid
        rows = tokens[j * shard:(j + 1) * shard]              # Alg. 1 l.5
        mbs = [rows[mu * microbatch:(mu + 1) * microbatch] for mu in range(m)]  # Alg. 2 l.2
        acts, dacts, caches = {}, {}, {}
        grads = [{n: np.zeros_like(v) for n, v in shards[i].items()} for i in range(g_inter)]
        last_b = [-1] * g_inter
        losses = []

        def on_forward(i, mu):
            inp = mbs[mu][:, :-1] if i == 0 else acts.pop((i - 1, mu))
            out, c = model.stage_forward(shards[i], cfg, i, g_inter, inp,
                                         labels=mbs[mu][:, 1:], m_total=m_total,
                                         loss_scale=loss_scale)
            caches[(i, mu)] = (c, inp)
            if i == g_inter - 1:
                losses.append(out)
            else:
                acts[(i, mu)] = out

        def on_backward(i, mu):
            assert mu == last_b[i] + 1, "backwards must run in ascending microbatch id (D-19)"
            last_b[i] = mu
            dout = 1.0 if i == g_inter - 1 else dacts.pop((i + 1, mu))
            c, _ = caches.pop((i, mu))
            dinp, g = model.stage_backward(shards[i], cfg, i, g_inter, c, dout)
            for n, v in g.items():
                if grad_accum == "half" and accumulates_in_half(n):   # D-38
                    grads[i][n] = round_half(grads[i][n] + round_half(v, half), half).astype(np.float64)
                else:
                    grads[i][n] += v
            if i > 0:
                dacts[(i, mu)] = dinp

        schedule.simulate(g_inter, m, policy=policy, on_forward=on_forward,
                          on_backward=on_backward, seed=seed)
        assert not caches and not acts and not dacts
        loss_total += sum(losses)
        per_replica.append(grads)
    # Alg. 1 l.13: all-reduce (SUM) over the column of each stage
    out = {}
    for i in range(g_inter):
        for n in shards[i]:
            acc = np.zeros_like(per_replica[0][i][n])
            for j in range(g_data):
                acc = acc + per_replica[j][i][n]
            out[n] = acc
    return loss_total, out
