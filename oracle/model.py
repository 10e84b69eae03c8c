"""GPT stage forward / backward and the pre-divided LM loss — oracle (test
infrastructure only; see oracle/__init__.py).

What it follows:

* The network is a "GPT-like transformer" for causal language modelling
  (Sec. VI-B).  The paper gives no layer equations, so the
  readings of SURVEY.md §8(c.2) apply (listed in DESIGN.md §2): D-1 GPT-2
  pre-LN block, learned token + position embeddings, 4h MLP, biases on every
  linear, final LN; D-2 QKV rows [q|k|v], heads contiguous; D-3 untied head,
  no bias; D-4 no dropout; D-5 tanh GeLU; D-6 LN eps 1e-5 biased variance;
  D-7 scale 1/sqrt(d); D-8 causal mask.
* A stage = nn_shard of contiguous layers;
  stage 0 also owns the embeddings and the last stage the final LN + head
  (D-21).  ``stage_forward`` is ``nn_shard.Forward`` and ``stage_backward`` is
  ``nn_shard.Backward`` of Alg. 2.
* Loss: token-mean cross entropy of the microbatch, multiplied by the loss
  scale S and pre-divided by the total number of microbatches in the batch
  (D-9, D-11), so that the SUM all-reduce of Alg. 1 l.13
  yields the mean gradient (D-10).

Everything is plain numpy in the dtype of the parameters (fp64 for pins).
Step order is the textbook order of each layer; there is no fusion.
Pins: tests/test_oracle_model.py (finite differences, torch-autograd fp64
cross-check, W_head = 0 closed form, causal invariance, s = 1 special case,
pre-division linearity).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

LN_EPS = 1e-5                      # D-6
GELU_C = 0.7978845608028654        # sqrt(2/pi), D-5
GELU_A = 0.044715                  # D-5


@dataclass(frozen=True)
class GPTConfig:
    n_layers: int
    hidden: int
    heads: int
    seq_len: int
    vocab: int

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


def layer_names(L: int):
    p = f"l{L}."
    return [p + n for n in ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o",
                            "ln2_g", "ln2_b", "w_fc1", "b_fc1", "w_fc2", "b_fc2")]


def stage_layers(cfg: GPTConfig, stage: int, n_stages: int):
    """Layers [i*l/G_inter, (i+1)*l/G_inter) — even contiguous split (D-21)."""
    per = cfg.n_layers // n_stages
    return list(range(stage * per, (stage + 1) * per))


def stage_param_names(cfg: GPTConfig, stage: int, n_stages: int):
    names = []
    if stage == 0:
        names += ["tok_emb", "pos_emb"]
    for L in stage_layers(cfg, stage, n_stages):
        names += layer_names(L)
    if stage == n_stages - 1:
        names += ["lnf_g", "lnf_b", "head_w"]
    return names


# ---------------------------------------------------------------- primitives
def ln_forward(z, g, b):
    """y = (z - mean) / sqrt(var_biased + eps) * g + b over the last axis (D-6)."""
    mu = z.mean(axis=-1, keepdims=True)
    var = ((z - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xhat = (z - mu) * rstd
    return xhat * g + b, (xhat, rstd)


def ln_backward(dy, g, cache):
    xhat, rstd = cache
    dxhat = dy * g
    n = xhat.shape[-1]
    dz = rstd * (dxhat - dxhat.sum(-1, keepdims=True) / n
                 - xhat * (dxhat * xhat).sum(-1, keepdims=True) / n)
    red = tuple(range(dy.ndim - 1))
    return dz, (dy * xhat).sum(axis=red), dy.sum(axis=red)


def gelu(x):
    """tanh-approximate GeLU (D-5)."""
    return 0.5 * x * (1.0 + np.tanh(GELU_C * (x + GELU_A * x ** 3)))


def gelu_grad(x):
    t = np.tanh(GELU_C * (x + GELU_A * x ** 3))
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * GELU_C * (1.0 + 3.0 * GELU_A * x * x)


def wgrad(dy, x):
    """Weight gradient sum_{b,s} dy[b,s,:]^T x[b,s,:] of a linear layer y = x W^T, evaluated
    as one matrix product (a library primitive; the same contraction as the einsum
    'bsn,bsk->nk', which numpy evaluates without BLAS)."""
    return dy.reshape(-1, dy.shape[-1]).T @ x.reshape(-1, x.shape[-1])


# ---------------------------------------------------------------- one layer
def layer_forward(p, L, cfg: GPTConfig, h):
    """Pre-LN transformer block (D-1): h [b, s, H] -> [b, s, H]."""
    n = f"l{L}."
    b, s, H = h.shape
    a, d = cfg.heads, cfg.head_dim
    u, c1 = ln_forward(h, p[n + "ln1_g"], p[n + "ln1_b"])
    qkv = u @ p[n + "w_qkv"].T + p[n + "b_qkv"]                    # [b, s, 3H]
    q = qkv[..., 0:H].reshape(b, s, a, d).transpose(0, 2, 1, 3)    # [b, a, s, d]  (D-2)
    k = qkv[..., H:2 * H].reshape(b, s, a, d).transpose(0, 2, 1, 3)
    v = qkv[..., 2 * H:3 * H].reshape(b, s, a, d).transpose(0, 2, 1, 3)
    scale = 1.0 / np.sqrt(d)                                        # D-7
    sc = (q @ k.transpose(0, 1, 3, 2)) * scale                      # [b, a, s, s]
    mask = np.triu(np.ones((s, s), dtype=bool), k=1)                # tau > t masked (D-8)
    sc = np.where(mask, -np.inf, sc)
    sc_max = sc.max(axis=-1, keepdims=True)
    e = np.exp(sc - sc_max)
    prob = e / e.sum(axis=-1, keepdims=True)
    o = (prob @ v).transpose(0, 2, 1, 3).reshape(b, s, H)          # merge heads
    h1 = h + o @ p[n + "w_o"].T + p[n + "b_o"]
    w, c2 = ln_forward(h1, p[n + "ln2_g"], p[n + "ln2_b"])
    pre = w @ p[n + "w_fc1"].T + p[n + "b_fc1"]
    act = gelu(pre)
    h2 = h1 + act @ p[n + "w_fc2"].T + p[n + "b_fc2"]
    cache = (u, c1, q, k, v, prob, o, w, c2, pre, act)
    return h2, cache


def layer_backward(p, L, cfg: GPTConfig, cache, dh2):
    n = f"l{L}."
    u, c1, q, k, v, prob, o, w, c2, pre, act = cache
    b, s, H = dh2.shape
    a, d = cfg.heads, cfg.head_dim
    red = (0, 1)
    gr = {}
    # h2 = h1 + act W2^T + b2
    gr[n + "w_fc2"] = wgrad(dh2, act)
    gr[n + "b_fc2"] = dh2.sum(axis=red)
    dact = dh2 @ p[n + "w_fc2"]
    dpre = dact * gelu_grad(pre)
    gr[n + "w_fc1"] = wgrad(dpre, w)
    gr[n + "b_fc1"] = dpre.sum(axis=red)
    dw = dpre @ p[n + "w_fc1"]
    dh1_ln, gr[n + "ln2_g"], gr[n + "ln2_b"] = ln_backward(dw, p[n + "ln2_g"], c2)
    dh1 = dh2 + dh1_ln
    # h1 = h + o Wo^T + bo
    gr[n + "w_o"] = wgrad(dh1, o)
    gr[n + "b_o"] = dh1.sum(axis=red)
    do = (dh1 @ p[n + "w_o"]).reshape(b, s, a, d).transpose(0, 2, 1, 3)
    scale = 1.0 / np.sqrt(d)
    dprob = do @ v.transpose(0, 1, 3, 2)
    dv = prob.transpose(0, 1, 3, 2) @ do
    dsc = prob * (dprob - (dprob * prob).sum(axis=-1, keepdims=True))   # softmax backward
    dsc = dsc * scale
    dq = dsc @ k
    dk = dsc.transpose(0, 1, 3, 2) @ q
    merge = lambda t: t.transpose(0, 2, 1, 3).reshape(b, s, H)
    dqkv = np.concatenate([merge(dq), merge(dk), merge(dv)], axis=-1)
    gr[n + "w_qkv"] = wgrad(dqkv, u)
    gr[n + "b_qkv"] = dqkv.sum(axis=red)
    du = dqkv @ p[n + "w_qkv"]
    dh_ln, gr[n + "ln1_g"], gr[n + "ln1_b"] = ln_backward(du, p[n + "ln1_g"], c1)
    return dh1 + dh_ln, gr


# ---------------------------------------------------------------- stages
def stage_forward(p, cfg: GPTConfig, stage: int, n_stages: int, inp, labels=None,
                  m_total: int = 1, loss_scale: float = 1.0):
    """nn_shard.Forward (Alg. 2 l.6/l.14/l.25).

    ``inp`` = int tokens [b, s] on stage 0, else the activation [b, s, H]
    received from stage i-1.  Returns (output, cache).  On the last stage the
    output is the pre-divided, scaled microbatch loss
    l_mu = S / M_total * mean_{b,t} CE (D-9, D-11) and the
    cache holds what Backward(1) needs; ``cache['ce_sum']`` is the unscaled
    CE sum for reporting."""
    caches = {}
    if stage == 0:
        tok = np.asarray(inp)
        s = tok.shape[1]
        h = p["tok_emb"][tok] + p["pos_emb"][None, :s]
        caches["tok"] = tok
    else:
        h = inp
    caches["layers"] = []
    for L in stage_layers(cfg, stage, n_stages):
        h, c = layer_forward(p, L, cfg, h)
        caches["layers"].append((L, c))
    if stage != n_stages - 1:
        return h, caches
    hf, cf = ln_forward(h, p["lnf_g"], p["lnf_b"])
    z = hf @ p["head_w"].T                                           # [b, s, V]
    zmax = z.max(axis=-1, keepdims=True)
    lse = np.log(np.exp(z - zmax).sum(axis=-1, keepdims=True)) + zmax
    y = np.asarray(labels)
    zy = np.take_along_axis(z, y[..., None], axis=-1)
    ce = (lse - zy)[..., 0]                                          # [b, s]
    ntok = ce.size
    loss = loss_scale / m_total * ce.mean()
    caches.update(hf=hf, cf=cf, z=z, lse=lse, y=y, ntok=ntok, m_total=m_total,
                  loss_scale=loss_scale, ce_sum=ce.sum())
    return loss, caches


def stage_backward(p, cfg: GPTConfig, stage: int, n_stages: int, caches, dout):
    """nn_shard.Backward (Alg. 2 l.15 ``Backward(1)`` on the last stage with
    dout = 1, l.22 with the received output-gradient otherwise).

    Returns (gradient w.r.t. the stage input or None on stage 0, grads)."""
    gr = {}
    if stage == n_stages - 1:
        z, lse, y = caches["z"], caches["lse"], caches["y"]
        soft = np.exp(z - lse)
        onehot = np.zeros_like(z)
        np.put_along_axis(onehot, y[..., None], 1.0, axis=-1)
        coef = dout * caches["loss_scale"] / (caches["m_total"] * caches["ntok"])
        dz = coef * (soft - onehot)
        gr["head_w"] = wgrad(dz, caches["hf"])
        dhf = dz @ p["head_w"]
        dh, gr["lnf_g"], gr["lnf_b"] = ln_backward(dhf, p["lnf_g"], caches["cf"])
    else:
        dh = dout
    for L, c in reversed(caches["layers"]):
        dh, g = layer_backward(p, L, cfg, c, dh)
        gr.update(g)
    if stage == 0:
        tok = caches["tok"]
        s = tok.shape[1]
        dtok = np.zeros_like(p["tok_emb"])
        np.add.at(dtok, tok.reshape(-1), dh.reshape(-1, dh.shape[-1]))
        gr["tok_emb"] = dtok
        dpos = np.zeros_like(p["pos_emb"])
        dpos[:s] = dh.sum(axis=0)
        gr["pos_emb"] = dpos
        return None, gr
    return dh, gr


def full_batch_loss_and_grads(p, cfg: GPTConfig, tokens, loss_scale: float = 1.0):
    """The plain definition the hybrid step reformulates:
    one sequential full-batch pass, loss = S * mean CE over all B*s tokens,
    exact gradient.  Equals Alg. 1 with G_inter = G_data = 1 and one
    microbatch."""
    tokens = np.asarray(tokens)
    loss, c = stage_forward(p, cfg, 0, 1, tokens[:, :-1], tokens[:, 1:], 1, loss_scale)
    _, g = stage_backward(p, cfg, 0, 1, c, 1.0)
    return loss, g
