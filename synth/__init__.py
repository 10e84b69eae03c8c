"""Seeded synthetic input generators shared by the oracle tests, the GPU parity
tests and ``bench.py``.

This module holds NONE of the method's arithmetic (no model math, no optimizer
math, no rounding mode of the method): it only draws numbers.  Both sides of
every parity test receive the exact same arrays from here, so the oracle
(``oracle/``) and the CUDA path (``paper_2110_13005_b200``) never have to share
code.  Input recipe (readings D-22/D-23):

* throughput tokens: uniform int32 in [0, V) from a counter-based splitmix64
  stream (cost of the step is value-independent);
* parity tokens: an order-1 Markov chain with 4 random successors per token,
  so the loss moves away from ln V when the model learns (D-23);
* weights: N(0, 0.02); W_o and W_2 use 0.02/sqrt(2l); LayerNorm gamma = 1,
  beta = 0, biases 0 (D-22).  ``parity=True`` perturbs gamma ~ 1 + N(0, 0.1)
  and beta/biases ~ N(0, 0.02) so every gradient is non-trivial.  All values
  are made bf16-representable by TRUNCATING the low 16 bits of the fp32
  pattern (D-15: theta16 == theta32 at step 0); truncation is deliberately not
  the method's round-to-nearest-even, which lives separately in each side.
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(seed: int, index: np.ndarray) -> np.ndarray:
    """Counter-based splitmix64: value for counter ``index`` under ``seed``."""
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) + (index.astype(np.uint64) + np.uint64(1))
             * np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_tokens(batch: int, seq_len: int, vocab: int, seed: int = 1234) -> np.ndarray:
    """int32 [batch, seq_len + 1] uniform token ids (inputs = [:, :s], labels = [:, 1:])."""
    n = batch * (seq_len + 1)
    z = splitmix64(seed, np.arange(n, dtype=np.uint64))
    return (z % np.uint64(vocab)).astype(np.int32).reshape(batch, seq_len + 1)


def markov_tokens(batch: int, seq_len: int, vocab: int, seed: int = 7,
                  successors: int = 4) -> np.ndarray:
    """int32 [batch, seq_len + 1] tokens from an order-1 Markov source.

    Each token has ``successors`` allowed next tokens drawn once per seed; the
    next token is a uniform choice among them."""
    rng = np.random.default_rng(seed)
    table = rng.integers(0, vocab, size=(vocab, successors), dtype=np.int64)
    out = np.empty((batch, seq_len + 1), dtype=np.int64)
    out[:, 0] = rng.integers(0, vocab, size=batch)
    choice = rng.integers(0, successors, size=(batch, seq_len))
    for t in range(seq_len):
        out[:, t + 1] = table[out[:, t], choice[:, t]]
    return out.astype(np.int32)


def _truncate_bf16(x: np.ndarray) -> np.ndarray:
    bits = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return (bits & np.uint32(0xFFFF0000)).view(np.float32)


def param_shapes(n_layers: int, hidden: int, seq_len: int, vocab: int):
    """Canonical (name, shape) list of the whole GPT, in flat order.

    Layout reading D-2 (QKV row blocks q|k|v, heads contiguous), D-3 (untied
    head, no bias), D-21 (embeddings on stage 0, final LN + head on the last
    stage).  Linear weights are [out, in] row-major."""
    h = hidden
    shapes = [("tok_emb", (vocab, h)), ("pos_emb", (seq_len, h))]
    for L in range(n_layers):
        p = f"l{L}."
        shapes += [
            (p + "ln1_g", (h,)), (p + "ln1_b", (h,)),
            (p + "w_qkv", (3 * h, h)), (p + "b_qkv", (3 * h,)),
            (p + "w_o", (h, h)), (p + "b_o", (h,)),
            (p + "ln2_g", (h,)), (p + "ln2_b", (h,)),
            (p + "w_fc1", (4 * h, h)), (p + "b_fc1", (4 * h,)),
            (p + "w_fc2", (h, 4 * h)), (p + "b_fc2", (h,)),
        ]
    shapes += [("lnf_g", (h,)), ("lnf_b", (h,)), ("head_w", (vocab, h))]
    return shapes


def init_params(n_layers: int, hidden: int, seq_len: int, vocab: int,
                seed: int = 42, parity: bool = True) -> dict:
    """fp32, bf16-representable initial weights (D-22), keyed by canonical name."""
    rng = np.random.default_rng(seed)
    out = {}
    proj_std = 0.02 / np.sqrt(2.0 * n_layers)
    for name, shape in param_shapes(n_layers, hidden, seq_len, vocab):
        leaf = name.split(".")[-1]
        if leaf.endswith("_g"):
            v = 1.0 + (rng.standard_normal(shape) * 0.1 if parity else 0.0)
            v = np.broadcast_to(np.asarray(v, dtype=np.float64), shape)
        elif leaf.endswith("_b") or leaf.startswith("b_"):
            v = rng.standard_normal(shape) * 0.02 if parity else np.zeros(shape)
        elif leaf in ("w_o", "w_fc2"):
            v = rng.standard_normal(shape) * proj_std
        else:
            v = rng.standard_normal(shape) * 0.02
        out[name] = _truncate_bf16(np.asarray(v, dtype=np.float32))
    return out


def adam_test_state(n: int, seed: int = 11):
    """Isolated-Adam parity data.

    theta ~ N(0, 0.02), m ~ N(0, 1e-3), v ~ |N(0, 1e-6)|, g ~ N(0, 1e-3)
    truncated to bf16, plus edge cases at the front: g = 0, v = 0, |g| >> 1,
    |g| ~ 1e-30 (flushes to a bf16 subnormal/zero), theta = 0."""
    rng = np.random.default_rng(seed)
    theta = (rng.standard_normal(n) * 0.02).astype(np.float32)
    m = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    v = np.abs(rng.standard_normal(n) * 1e-6).astype(np.float32)
    g = _truncate_bf16((rng.standard_normal(n) * 1e-3).astype(np.float32))
    k = min(n, 8)
    edge_g = np.array([0.0, 0.0, 1e3, -1e3, 1e-30, -1e-30, 5.0, 0.0], dtype=np.float32)[:k]
    g[:k] = _truncate_bf16(edge_g)
    v[:k] = np.array([0.0, 1e-6, 0.0, 1.0, 0.0, 0.0, 0.0, 0.0], dtype=np.float32)[:k]
    m[:k] = np.array([0.0, 0.0, 0.0, 0.0, 0.0, 1e-3, 0.0, 0.0], dtype=np.float32)[:k]
    theta[:k] = np.array([0.5, -0.5, 0.0, 1.0, 0.02, 0.0, -1.0, 0.0], dtype=np.float32)[:k]
    return theta, m, v, g


def mixed_batch(distinct: np.ndarray, batch: int, seed: int = 5):
    """A full-size parity batch built from a few distinct sequences without a period.

    Row r of the batch is ``distinct[assign[r]]`` with ``assign`` drawn uniformly (seeded),
    every distinct sequence used at least once.  The exact batch gradient is then the
    multiplicity-weighted sum of the per-sequence gradients, which the oracle computes from
    the distinct sequences alone; because the assignment has no period, a row, sample or
    microbatch offset error changes the multiset of rows the GPU reads and hence the result
    (a tiled [s0, s1, s0, s1, ...] batch hides every offset error by an even count).
    Returns (tokens int32 [batch, s + 1], counts int64 [n_distinct])."""
    n = distinct.shape[0]
    assert batch >= n
    rng = np.random.default_rng(seed)
    assign = np.concatenate([np.arange(n), rng.integers(0, n, size=batch - n)])
    rng.shuffle(assign)
    counts = np.bincount(assign, minlength=n).astype(np.int64)
    return np.ascontiguousarray(distinct[assign]).astype(np.int32), counts
