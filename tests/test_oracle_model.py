"""Pins for oracle/model.py (SURVEY.md §8(c.3) pins 1-6).

Each test ties the oracle to something other than itself: central finite
differences (brute force), an independent torch-autograd fp64 re-implementation
(library routine), closed forms (W_head = 0), invariants (causality,
pre-division linearity) and a special case (s = 1)."""
import math

import numpy as np
import pytest

from oracle import model
from synth import init_params, markov_tokens

MICRO = model.GPTConfig(n_layers=2, hidden=8, heads=2, seq_len=4, vocab=11)
TINY = model.GPTConfig(n_layers=2, hidden=64, heads=2, seq_len=32, vocab=256)


def params64(cfg, seed=42):
    p = init_params(cfg.n_layers, cfg.hidden, cfg.seq_len, cfg.vocab, seed=seed, parity=True)
    return {k: v.astype(np.float64) for k, v in p.items()}


def loss_of(p, cfg, tok):
    return model.full_batch_loss_and_grads(p, cfg, tok)[0]


def test_finite_differences_every_parameter_micro():
    """Pin 1: central FD in fp64 for EVERY parameter of a micro GPT."""
    cfg = MICRO
    p = params64(cfg)
    tok = markov_tokens(2, cfg.seq_len, cfg.vocab, seed=3)
    _, g = model.full_batch_loss_and_grads(p, cfg, tok)
    worst = 0.0
    for name, val in p.items():
        flat = val.reshape(-1)
        for idx in range(flat.size):
            old = flat[idx]
            step = 1e-5 * max(1.0, abs(old))
            flat[idx] = old + step
            lp = loss_of(p, cfg, tok)
            flat[idx] = old - step
            lm = loss_of(p, cfg, tok)
            flat[idx] = old
            fd = (lp - lm) / (2 * step)
            ad = g[name].reshape(-1)[idx]
            err = abs(fd - ad)
            bound = 1e-6 * max(abs(fd), abs(ad)) + 1e-9
            worst = max(worst, err / bound)
            assert err <= bound, (name, idx, fd, ad)
    assert worst <= 1.0


def test_finite_differences_sampled_tiny():
    """Pin 1 on the BASELINE tiny config (l 2, h 64, a 2, s 32, V 256): 6 random
    entries of every tensor."""
    cfg = TINY
    p = params64(cfg)
    tok = markov_tokens(2, cfg.seq_len, cfg.vocab, seed=5)
    _, g = model.full_batch_loss_and_grads(p, cfg, tok)
    rng = np.random.default_rng(0)
    for name, val in p.items():
        flat = val.reshape(-1)
        if name == "tok_emb":   # only rows that occur carry gradient; test those + one absent
            cand = np.unique(tok[:, :-1])[:4] * cfg.hidden + 3
            idxs = list(cand) + [int(np.setdiff1d(np.arange(cfg.vocab), tok)[0]) * cfg.hidden]
        else:
            idxs = rng.choice(flat.size, size=min(6, flat.size), replace=False)
        for idx in idxs:
            old = flat[idx]
            step = 1e-5 * max(1.0, abs(old))
            flat[idx] = old + step
            lp = loss_of(p, cfg, tok)
            flat[idx] = old - step
            lm = loss_of(p, cfg, tok)
            flat[idx] = old
            fd = (lp - lm) / (2 * step)
            ad = g[name].reshape(-1)[idx]
            assert abs(fd - ad) <= 1e-6 * max(abs(fd), abs(ad)) + 1e-9, (name, idx, fd, ad)


def _torch_gpt_loss(tp, cfg, tok):
    """Independent torch fp64 GPT (readings D-1..D-9) built from torch library
    ops (layer_norm, softmax, gelu(tanh), cross_entropy) — test-only."""
    import torch
    import torch.nn.functional as F
    b, s = tok.shape[0], tok.shape[1] - 1
    x = torch.as_tensor(tok[:, :-1], dtype=torch.long)
    y = torch.as_tensor(tok[:, 1:], dtype=torch.long)
    H, a = cfg.hidden, cfg.heads
    d = H // a
    h = tp["tok_emb"][x] + tp["pos_emb"][:s]
    mask = torch.ones(s, s, dtype=torch.bool).triu(1)
    for L in range(cfg.n_layers):
        n = f"l{L}."
        u = F.layer_norm(h, (H,), tp[n + "ln1_g"], tp[n + "ln1_b"], eps=1e-5)
        qkv = F.linear(u, tp[n + "w_qkv"], tp[n + "b_qkv"])
        q, k, v = qkv.split(H, dim=-1)
        q, k, v = (t.view(b, s, a, d).transpose(1, 2) for t in (q, k, v))
        att = (q @ k.transpose(-1, -2)) / math.sqrt(d)
        att = att.masked_fill(mask, float("-inf")).softmax(-1)
        o = (att @ v).transpose(1, 2).reshape(b, s, H)
        h = h + F.linear(o, tp[n + "w_o"], tp[n + "b_o"])
        w = F.layer_norm(h, (H,), tp[n + "ln2_g"], tp[n + "ln2_b"], eps=1e-5)
        f = F.gelu(F.linear(w, tp[n + "w_fc1"], tp[n + "b_fc1"]), approximate="tanh")
        h = h + F.linear(f, tp[n + "w_fc2"], tp[n + "b_fc2"])
    hf = F.layer_norm(h, (H,), tp["lnf_g"], tp["lnf_b"], eps=1e-5)
    z = F.linear(hf, tp["head_w"])
    return F.cross_entropy(z.reshape(-1, cfg.vocab), y.reshape(-1))


@pytest.mark.parametrize("cfg", [MICRO, TINY])
def test_torch_autograd_fp64_crosscheck(cfg):
    """Pin 5: loss and every gradient vs torch autograd fp64, rel <= 1e-12."""
    import torch
    p = params64(cfg, seed=9)
    tok = markov_tokens(4, cfg.seq_len, cfg.vocab, seed=11)
    loss, g = model.full_batch_loss_and_grads(p, cfg, tok)
    tp = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in p.items()}
    tl = _torch_gpt_loss(tp, cfg, tok)
    tl.backward()
    assert abs(loss - tl.item()) <= 1e-12 * abs(tl.item())
    for k in p:
        ref = tp[k].grad.numpy()
        num = np.linalg.norm(g[k] - ref)
        den = np.linalg.norm(ref)
        assert num <= 1e-12 * den + 1e-300, (k, num, den)


def test_zero_head_closed_form():
    """Pin 2: W_head = 0 => z = 0 => loss/S = ln V exactly, every non-head
    gradient is 0, and grad W_head = dz^T LN_f(h) with dz = S (1/V - onehot) / (M_total b s)."""
    cfg = TINY
    p = params64(cfg)
    p["head_w"][:] = 0.0
    tok = markov_tokens(2, cfg.seq_len, cfg.vocab, seed=2)
    S, m_total = 4.0, 2
    loss, c = model.stage_forward(p, cfg, 0, 1, tok[:, :-1], tok[:, 1:], m_total, S)
    assert loss * m_total / S == pytest.approx(math.log(256), rel=1e-15, abs=0)
    assert math.log(256) == 5.545177444479562
    _, g = model.stage_backward(p, cfg, 0, 1, c, 1.0)
    for k, v in g.items():
        if k != "head_w":
            assert np.all(v == 0.0), k
    b, s = tok.shape[0], cfg.seq_len
    dz = np.full((b, s, cfg.vocab), 1.0 / cfg.vocab)
    dz[np.arange(b)[:, None], np.arange(s)[None, :], tok[:, 1:]] -= 1.0
    dz *= S / (m_total * b * s)
    expect = np.einsum("bsv,bsk->vk", dz, c["hf"])
    np.testing.assert_allclose(g["head_w"], expect, rtol=1e-13, atol=1e-18)


def test_causal_mask_invariance():
    """Pin 3: changing tokens at positions > t leaves logits z[:, :t+1] bit-identical."""
    cfg = TINY
    p = params64(cfg)
    tok = markov_tokens(2, cfg.seq_len, cfg.vocab, seed=4)
    t = 13
    _, c1 = model.stage_forward(p, cfg, 0, 1, tok[:, :-1], tok[:, 1:])
    tok2 = tok.copy()
    tok2[:, t + 1:] = (tok2[:, t + 1:] + 17) % cfg.vocab
    _, c2 = model.stage_forward(p, cfg, 0, 1, tok2[:, :-1], tok2[:, 1:])
    assert np.array_equal(c1["z"][:, :t + 1], c2["z"][:, :t + 1])
    assert not np.array_equal(c1["z"][:, t + 1:], c2["z"][:, t + 1:])


def test_single_position_attention_is_v():
    """Pin 4: s = 1 => softmax weight 1 => attention output o = v."""
    cfg = model.GPTConfig(n_layers=1, hidden=16, heads=4, seq_len=1, vocab=13)
    p = params64(cfg)
    tok = markov_tokens(3, 1, cfg.vocab, seed=1)
    _, c = model.stage_forward(p, cfg, 0, 1, tok[:, :-1], tok[:, 1:])
    (_, lc), = c["layers"]
    u, c1, q, k, v, prob, o, *_ = lc
    assert np.all(prob == 1.0)
    merged_v = v.transpose(0, 2, 1, 3).reshape(o.shape)
    assert np.array_equal(o, merged_v)


def test_predivision_linearity():
    """Pin 6: doubling M_total halves the loss and every gradient exactly."""
    cfg = TINY
    p = params64(cfg)
    tok = markov_tokens(2, cfg.seq_len, cfg.vocab, seed=6)
    l1, c1 = model.stage_forward(p, cfg, 0, 1, tok[:, :-1], tok[:, 1:], 2, 1.0)
    l2, c2 = model.stage_forward(p, cfg, 0, 1, tok[:, :-1], tok[:, 1:], 4, 1.0)
    assert l2 == l1 / 2
    _, g1 = model.stage_backward(p, cfg, 0, 1, c1, 1.0)
    _, g2 = model.stage_backward(p, cfg, 0, 1, c2, 1.0)
    for k in g1:
        assert np.array_equal(g2[k], g1[k] / 2), k
