"""Kernel-level parity of the fused causal attention (K2, include/axonn.h axonn_k_attn_fwd)
against the plain definition softmax_causal(alpha Q K^T) V in fp64 on the SAME bf16-rounded
Q, K, V (readings D-7, D-8).  Shapes cover the tiny config, the 1.3B
attention (s 512, d 128), a ragged sequence length, and the padded 12B / 24B head widths
(d 188 -> dp 192, d 176)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2110_13005_b200 import _lib
    return _lib.load()


def make_qkv(b, heads, s, d, dp, seed):
    import torch
    rng = np.random.default_rng(seed)
    x = np.zeros((b * s, 3, heads, dp), np.float32)
    x[..., :d] = rng.standard_normal((b * s, 3, heads, d)) * 1.5
    t = torch.from_numpy(x.reshape(b * s, 3 * heads * dp)).to(torch.bfloat16).cuda()
    return t, t.float().cpu().numpy().astype(np.float64).reshape(b, s, 3, heads, dp)


def reference(x, d, alpha):
    b, s, _, heads, dp = x.shape
    o = np.zeros((b, s, heads, d))
    lse = np.zeros((b, heads, s))
    mask = np.tril(np.ones((s, s), bool))
    for i in range(b):
        for n in range(heads):
            q, k, v = x[i, :, 0, n, :d], x[i, :, 1, n, :d], x[i, :, 2, n, :d]
            z = alpha * np.log2(np.e) * (q @ k.T)
            z = np.where(mask, z, -np.inf)
            m = z.max(axis=1, keepdims=True)
            e = np.exp2(z - m)
            ssum = e.sum(axis=1, keepdims=True)
            o[i, :, n] = (e / ssum) @ v
            lse[i, n] = (m + np.log2(ssum))[:, 0]
    return o, lse


@pytest.mark.parametrize("b,heads,s,d,dp", [(2, 2, 32, 32, 32), (1, 4, 512, 128, 128),
                                            (2, 3, 200, 64, 64), (1, 2, 512, 188, 192),
                                            (1, 2, 384, 176, 176), (8, 2, 512, 128, 128),
                                            (1, 2, 1024, 128, 128), (1, 2, 700, 10, 16),
                                            (2, 1, 520, 188, 192)])
def test_attn_fwd_matches_definition(lib, b, heads, s, d, dp):
    """Streamed-key forward at any s: one, two and several 256-query units, ragged tails (the
    second tile of the last unit partly or wholly past s), 64 / 128 / 192-wide padded heads."""
    run_fwd(lib, b, heads, s, d, dp, make_qkv(b, heads, s, d, dp, seed=s + d))


def test_attn_fwd_rescale_path(lib):
    """Keys whose scores grow along the sequence (k_t scaled by 1 + 6 t / s): a row's running
    max rises by far more than the lazy-rescale threshold (2^8) from block to block, so the
    online softmax takes its rescale path (l and the O row multiplied by exp2(m - m'))."""
    import torch
    b, heads, s, d, dp = 1, 2, 512, 128, 128
    rng = np.random.default_rng(5)
    x = np.zeros((b * s, 3, heads, dp), np.float32)
    x[..., :d] = rng.standard_normal((b * s, 3, heads, d)) * 1.5
    x[:, 1] *= (1.0 + 6.0 * np.arange(b * s) / s)[:, None, None]
    t = torch.from_numpy(x.reshape(b * s, 3 * heads * dp)).to(torch.bfloat16).cuda()
    run_fwd(lib, b, heads, s, d, dp, (t, t.float().cpu().numpy().astype(np.float64).reshape(b, s, 3, heads, dp)))


def run_fwd(lib, b, heads, s, d, dp, made):
    import torch
    qkv, x = made
    h = heads * d
    o = torch.full((b * s, h), float("nan"), dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros(b * heads * s, dtype=torch.float32, device="cuda")
    alpha = 1.0 / np.sqrt(d)
    rc = lib.axonn_k_attn_fwd(C.c_void_p(qkv.data_ptr()), 3 * heads * dp, b, heads, s, d, dp,
                              C.c_float(alpha), C.c_void_p(o.data_ptr()), h,
                              C.c_void_p(lse.data_ptr()), None)
    assert rc == 0, rc
    torch.cuda.synchronize()
    o_ref, lse_ref = reference(x, d, alpha)
    out = o.float().cpu().numpy().astype(np.float64).reshape(b, s, heads, d)
    assert np.isfinite(out).all()
    err = np.linalg.norm(out - o_ref) / np.linalg.norm(o_ref)
    cos = (out * o_ref).sum() / (np.linalg.norm(out) * np.linalg.norm(o_ref))
    assert err < 1e-2 and cos > 0.9999, (err, cos)
    l = lse.cpu().numpy().astype(np.float64).reshape(b, heads, s)
    assert np.abs(l - lse_ref).max() < 2e-3


def reference_grads(x, dout, d, alpha):
    """Plain definition: P = softmax_causal(alpha Q K^T); dV = P^T dO; dP = dO V^T;
    dS = P * (dP - rowsum(P * dP)); dQ = alpha dS K; dK = alpha dS^T Q."""
    b, s, _, heads, dp = x.shape
    g = np.zeros((b, s, 3, heads, d))
    mask = np.tril(np.ones((s, s), bool))
    for i in range(b):
        for n in range(heads):
            q, k, v = x[i, :, 0, n, :d], x[i, :, 1, n, :d], x[i, :, 2, n, :d]
            do = dout[i, :, n, :d]
            z = np.where(mask, alpha * (q @ k.T), -np.inf)
            P = np.exp(z - z.max(axis=1, keepdims=True))
            P /= P.sum(axis=1, keepdims=True)
            dP = do @ v.T
            dS = P * (dP - (P * dP).sum(axis=1, keepdims=True))
            g[i, :, 0, n] = alpha * dS @ k
            g[i, :, 1, n] = alpha * dS.T @ q
            g[i, :, 2, n] = P.T @ do
    return g


@pytest.mark.parametrize("b,heads,s,d,dp", [(2, 2, 32, 32, 32), (1, 4, 512, 128, 128),
                                            (2, 3, 200, 64, 64), (1, 2, 512, 188, 192),
                                            (1, 2, 384, 176, 176), (8, 2, 512, 128, 128),
                                            (2, 4, 256, 188, 192), (1, 8, 96, 176, 176)])
def test_attn_bwd_matches_definition(lib, b, heads, s, d, dp):
    import torch
    qkv, x = make_qkv(b, heads, s, d, dp, seed=3 * s + d)
    h = heads * d
    rng = np.random.default_rng(s)
    dpad = np.zeros((b * s, heads, dp), np.float32)
    dpad[..., :d] = rng.standard_normal((b * s, heads, d))
    dO = torch.from_numpy(dpad.reshape(b * s, heads * dp)).to(torch.bfloat16).cuda()
    o = torch.empty((b * s, h), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(b * heads * s, dtype=torch.float32, device="cuda")
    dbuf = torch.empty(b * heads * s, dtype=torch.float32, device="cuda")
    dqkv = torch.full((b * s, 3 * h), float("nan"), dtype=torch.bfloat16, device="cuda")
    alpha = 1.0 / np.sqrt(d)
    P = C.c_void_p
    assert lib.axonn_k_attn_fwd(P(qkv.data_ptr()), 3 * heads * dp, b, heads, s, d, dp, C.c_float(alpha),
                                P(o.data_ptr()), h, P(lse.data_ptr()), None) == 0
    rc = lib.axonn_k_attn_bwd(P(qkv.data_ptr()), 3 * heads * dp, P(dO.data_ptr()), P(o.data_ptr()), h,
                              P(lse.data_ptr()), P(dbuf.data_ptr()), b, heads, s, d, dp, C.c_float(alpha),
                              P(dqkv.data_ptr()), 3 * h, None)
    assert rc == 0, rc
    torch.cuda.synchronize()
    dout = dO.float().cpu().numpy().astype(np.float64).reshape(b, s, heads, dp)
    ref = reference_grads(x, dout, d, alpha)
    got = dqkv.float().cpu().numpy().astype(np.float64).reshape(b, s, 3, heads, d)
    assert np.isfinite(got).all()
    res = {}
    for w, name in enumerate(("dQ", "dK", "dV")):
        g, r = got[:, :, w], ref[:, :, w]
        err = np.linalg.norm(g - r) / np.linalg.norm(r)
        cos = (g * r).sum() / (np.linalg.norm(g) * np.linalg.norm(r))
        res[name] = (err, cos)
    D = dbuf.cpu().numpy().astype(np.float64).reshape(b, heads, s)
    o_h = o.float().cpu().numpy().astype(np.float64).reshape(b, s, heads, d)
    D_ref = np.einsum("bsnd,bsnd->bns", dout[..., :d], o_h)
    res["D"] = float(np.abs(D - D_ref).max())
    print(res)
    for name in ("dQ", "dK", "dV"):
        err, cos = res[name]
        assert err < 2e-2 and cos > 0.9995, (name, res)
    # bitwise reproducible (one writer per element, no atomics)
    first = dqkv.clone()
    assert lib.axonn_k_attn_bwd(P(qkv.data_ptr()), 3 * heads * dp, P(dO.data_ptr()), P(o.data_ptr()), h,
                                P(lse.data_ptr()), P(dbuf.data_ptr()), b, heads, s, d, dp, C.c_float(alpha),
                                P(dqkv.data_ptr()), 3 * h, None) == 0
    torch.cuda.synchronize()
    assert torch.equal(first, dqkv)
