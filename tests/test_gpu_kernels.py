"""Kernel-level parity (T2): K1 tcgen05 GEMM and K9 AdamW through the C-ABI.

References: numpy fp64 products of the SAME bf16-rounded inputs (a matmul is a
library primitive, ③) and the fp32 oracle AdamW (bit-exact by design, D-14)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2110_13005_b200 import _lib
    return _lib.load()


def torch():
    import torch as t
    return t


def dev_bf16(x):
    t = torch()
    return t.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(t.bfloat16).cuda()


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


def gemm(lib, **kw):
    from paper_2110_13005_b200._lib import GemmArgs
    a = GemmArgs()
    defaults = dict(Z=1, Z1=1, a_s1=0, a_s2=0, b_s1=0, b_s2=0, c_s1=0, c_s2=0, alpha=1.0)
    defaults.update(kw)
    for k, v in defaults.items():
        if hasattr(v, "data_ptr"):
            v = v.data_ptr()
        setattr(a, k, v)
    rc = lib.axonn_k_gemm(C.byref(a), None)
    assert rc == 0, rc
    torch().cuda.synchronize()


def rel(x, ref):
    return np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-30)


def cos(x, ref):
    return float((x * ref).sum() / (np.linalg.norm(x) * np.linalg.norm(ref) + 1e-300))


RNG = np.random.default_rng(1234)


VARIANTS = pytest.mark.parametrize("variant", [1, 2, 3])


@VARIANTS
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 520, 200), (1024, 768, 1024),
                                   (4096, 2048, 2048), (77, 16, 8), (640, 384, 72),
                                   (1024, 96, 320)])   # variant 2: the 256 x 128 pair tile
def test_gemm_forward_bias_resid(lib, M, N, K, variant):
    t = torch()
    A = dev_bf16(RNG.standard_normal((M, K)))
    B = dev_bf16(RNG.standard_normal((N, K)) * 0.05)
    bias = dev_bf16(RNG.standard_normal(N))
    res = dev_bf16(RNG.standard_normal((M, N)))
    Cd = t.empty((M, N), dtype=t.bfloat16, device="cuda")
    gemm(lib, M=M, N=N, K=K, A=A, lda=K, a_mn=0, B=B, ldb=K, b_mn=0, C=Cd, ldc=N, epi=0,
         bias=bias, resid=res, ld_resid=N, variant=variant)
    ref = host(A) @ host(B).T + host(bias) + host(res)
    out = host(Cd)
    assert rel(out, ref) < 1e-2 and cos(out, ref) > 0.9999


@VARIANTS
@pytest.mark.parametrize("M,N,K", [(256, 200, 384), (4096, 2048, 8192), (130, 72, 64),
                                   (520, 328, 136)])
def test_gemm_dgrad_b_mn_major(lib, M, N, K, variant):
    """dX = dY W: B stored [K][N] (MN-major)."""
    t = torch()
    A = dev_bf16(RNG.standard_normal((M, K)))
    W = dev_bf16(RNG.standard_normal((K, N)) * 0.05)
    Cd = t.empty((M, N), dtype=t.bfloat16, device="cuda")
    gemm(lib, M=M, N=N, K=K, A=A, lda=K, a_mn=0, B=W, ldb=N, b_mn=1, C=Cd, ldc=N, epi=0,
         variant=variant)
    ref = host(A) @ host(W)
    out = host(Cd)
    assert rel(out, ref) < 1e-2 and cos(out, ref) > 0.9999


@VARIANTS
@pytest.mark.parametrize("M,N,K", [(192, 320, 500), (2048, 8192, 4096), (64, 136, 40),
                                   (392, 264, 128)])
def test_gemm_wgrad_both_mn_major_f32_accumulate(lib, M, N, K, variant):
    """dW (+)= dY^T X: A stored [K][M], B stored [K][N]; fp32 output, accumulate."""
    t = torch()
    dY = dev_bf16(RNG.standard_normal((K, M)))
    X = dev_bf16(RNG.standard_normal((K, N)))
    Cd = t.zeros((M, N), dtype=t.float32, device="cuda")
    for acc in (0, 1):
        gemm(lib, M=M, N=N, K=K, A=dY, lda=M, a_mn=1, B=X, ldb=N, b_mn=1, C=Cd, ldc=N, epi=3,
             accumulate=acc, variant=variant)
    ref = 2 * host(dY).T @ host(X)
    out = Cd.cpu().numpy().astype(np.float64)
    assert rel(out, ref) < 1e-5


@VARIANTS
def test_gemm_gelu_and_dgelu(lib, variant):
    t = torch()
    M, N, K = 256, 512, 192
    A = dev_bf16(RNG.standard_normal((M, K)))
    B = dev_bf16(RNG.standard_normal((N, K)) * 0.1)
    bias = dev_bf16(RNG.standard_normal(N) * 0.1)
    out = t.empty((M, N), dtype=t.bfloat16, device="cuda")
    pre = t.empty((M, N), dtype=t.bfloat16, device="cuda")
    gemm(lib, M=M, N=N, K=K, A=A, lda=K, B=B, ldb=K, C=out, ldc=N, epi=1, bias=bias, aux=pre,
         ld_aux=N, variant=variant)
    pre_ref = host(A) @ host(B).T + host(bias)
    assert rel(host(pre), pre_ref) < 1e-2
    p = host(pre)
    c = 0.7978845608028654
    gelu = 0.5 * p * (1 + np.tanh(c * (p + 0.044715 * p ** 3)))
    assert rel(host(out), gelu) < 1e-2
    # DGELU: out2 = (A B^T) * gelu'(pre)
    out2 = t.empty((M, N), dtype=t.bfloat16, device="cuda")
    gemm(lib, M=M, N=N, K=K, A=A, lda=K, B=B, ldb=K, C=out2, ldc=N, epi=2, aux=pre, ld_aux=N,
         variant=variant)
    th = np.tanh(c * (p + 0.044715 * p ** 3))
    dg = 0.5 * (1 + th) + 0.5 * p * (1 - th * th) * c * (1 + 3 * 0.044715 * p * p)
    ref2 = (host(A) @ host(B).T) * dg
    assert rel(host(out2), ref2) < 1e-2


@VARIANTS
def test_gemm_batched_attention_shapes(lib, variant):
    """S = Q K^T over (sample, head) from the packed [b*s, 3h] QKV layout via
    4-D TMA maps; causal modes 1 (skip upper tiles), 2 (k < m0+128), 3 (k >= m0)."""
    t = torch()
    b, s, a, d = 2, 384, 3, 64
    h = a * d
    qkv = dev_bf16(RNG.standard_normal((b * s, 3 * h)))
    Q = host(qkv)[:, :h].reshape(b, s, a, d).transpose(0, 2, 1, 3)
    Kt = host(qkv)[:, h:2 * h].reshape(b, s, a, d).transpose(0, 2, 1, 3)
    S = t.full((b, a, s, s), float("nan"), dtype=t.float32, device="cuda")
    gemm(lib, M=s, N=s, K=d, Z=b * a, Z1=a,
         A=qkv, lda=3 * h, a_s1=d, a_s2=s * 3 * h, a_mn=0,
         B=qkv[:, h:], ldb=3 * h, b_s1=d, b_s2=s * 3 * h, b_mn=0,
         C=S, ldc=s, c_s1=s * s, c_s2=a * s * s, epi=3, causal=1, alpha=0.5, variant=variant)
    ref = 0.5 * Q @ Kt.transpose(0, 1, 3, 2)
    got = S.cpu().numpy()
    low = np.tril(np.ones((s, s), dtype=bool))
    assert rel(got[..., low], ref[..., low]) < 1e-5
    # PV: O[q, e] = sum_{k <= q-block} P[q, k] V[k, e] with P lower-triangular
    P = np.tril(RNG.standard_normal((b, a, s, s)))
    Pd = dev_bf16(P)
    O = t.zeros((b * s, h), dtype=t.bfloat16, device="cuda")
    gemm(lib, M=s, N=d, K=s, Z=b * a, Z1=a,
         A=Pd, lda=s, a_s1=s * s, a_s2=a * s * s, a_mn=0,
         B=qkv[:, 2 * h:], ldb=3 * h, b_s1=d, b_s2=s * 3 * h, b_mn=1,
         C=O, ldc=h, c_s1=d, c_s2=s * h, epi=0, causal=2)
    V = host(qkv)[:, 2 * h:].reshape(b, s, a, d).transpose(0, 2, 1, 3)
    refO = (host(Pd) @ V).transpose(0, 2, 1, 3).reshape(b * s, h)
    assert rel(host(O), refO) < 1e-2
    # dK = dS^T Q with dS lower-triangular: A = dS^T (MN-major), B = Q^T (MN-major), causal 3
    dK = t.zeros((b * s, h), dtype=t.bfloat16, device="cuda")
    gemm(lib, M=s, N=d, K=s, Z=b * a, Z1=a,
         A=Pd, lda=s, a_s1=s * s, a_s2=a * s * s, a_mn=1,
         B=qkv, ldb=3 * h, b_s1=d, b_s2=s * 3 * h, b_mn=1,
         C=dK, ldc=h, c_s1=d, c_s2=s * h, epi=0, causal=3)
    refK = (host(Pd).transpose(0, 1, 3, 2) @ Q).transpose(0, 2, 1, 3).reshape(b * s, h)
    assert rel(host(dK), refK) < 1e-2


def test_gemm_column_remap_and_nvalid(lib):
    """Columns c -> (c / 5) * 8 + c % 5 (head padding layout); n_valid cut."""
    t = torch()
    M, N, K = 130, 40, 64
    A = dev_bf16(RNG.standard_normal((M, K)))
    B = dev_bf16(RNG.standard_normal((N, K)))
    Cd = t.zeros((M, 64), dtype=t.bfloat16, device="cuda")
    gemm(lib, M=M, N=N, K=K, A=A, lda=K, B=B, ldb=K, C=Cd, ldc=64, epi=0, col_group_in=5,
         col_group_out=8)
    ref = host(A) @ host(B).T
    out = host(Cd)
    for c in range(N):
        dc = (c // 5) * 8 + c % 5
        assert rel(out[:, dc], ref[:, c]) < 1e-2
    pad = [dc for dc in range(64) if dc % 8 >= 5]
    assert np.all(out[:, pad] == 0)
    Cd2 = t.zeros((M, N), dtype=t.bfloat16, device="cuda")
    gemm(lib, M=M, N=N, K=K, A=A, lda=K, B=B, ldb=K, C=Cd2, ldc=N, epi=0, n_valid=37)
    o2 = host(Cd2)
    assert np.all(o2[:, 37:] == 0) and rel(o2[:, :37], ref[:, :37]) < 1e-2


@pytest.mark.parametrize("M,groups,d,dp,K", [(512, 12, 188, 192, 256), (300, 7, 120, 128, 64),
                                              (4096, 72, 188, 192, 512)])
def test_gemm_column_remap_tma_epilogue(lib, M, groups, d, dp, K):
    """The remapped TMA-store epilogue (3-D map, two clipped stores where a 64-column box
    crosses a group edge; the QKV forward / attention-output dgrad at d != dp, D-7): same bf16
    values as the thread-store epilogue (variant 3), padding columns untouched, vs numpy."""
    t = torch()
    N = groups * d
    A = dev_bf16(RNG.standard_normal((M, K)))
    B = dev_bf16(RNG.standard_normal((N, K)) * 0.05)
    bias = dev_bf16(RNG.standard_normal(N))
    outs = []
    for variant in (0, 3):
        Cd = t.full((M, groups * dp), 7.0, dtype=t.bfloat16, device="cuda")
        gemm(lib, M=M, N=N, K=K, A=A, lda=K, B=B, ldb=K, C=Cd, ldc=groups * dp, epi=0,
             bias=bias, col_group_in=d, col_group_out=dp, variant=variant)
        outs.append(host(Cd))
    assert np.array_equal(outs[0], outs[1])
    out = outs[0].reshape(M, groups, dp)
    assert np.all(out[:, :, d:] == 7.0)
    ref = (host(A) @ host(B).T + host(bias)).reshape(M, groups, d)
    assert rel(out[:, :, :d], ref) < 1e-2


@pytest.mark.parametrize("variant", [0, 3])
@pytest.mark.parametrize("M,N,K", [(512, 768, 1024), (304, 200, 520), (2048, 4096, 512)])
def test_gemm_wgrad_half_accumulate(lib, M, N, K, variant):
    """grad_accum_fp32 = 0 (reading D-38): the wgrad GEMM adds its product into a half
    gradient, C <- RN(C + RN(dY^T X)).  Bit for bit against that definition evaluated on the
    host from the same kernel's fp32 product (epi 3 into a zeroed fp32 C), for the TMA
    reduce-add epilogue (variant 0) and the thread-store one (variant 3)."""
    from oracle.bf16 import round_bf16
    t = torch()
    dY = dev_bf16(RNG.standard_normal((K, M)))    # MN-major operands as in the engine's wgrad
    X = dev_bf16(RNG.standard_normal((K, N)))
    F = t.zeros((M, N), dtype=t.float32, device="cuda")
    gemm(lib, M=M, N=N, K=K, A=dY, lda=M, a_mn=1, B=X, ldb=N, b_mn=1, C=F, ldc=N, epi=3,
         accumulate=0, variant=variant)
    v = F.cpu().numpy()
    C0 = RNG.standard_normal((M, N)) * np.sqrt(K)
    Cd = dev_bf16(C0)
    c0 = Cd.float().cpu().numpy().astype(np.float64)
    gemm(lib, M=M, N=N, K=K, A=dY, lda=M, a_mn=1, B=X, ldb=N, b_mn=1, C=Cd, ldc=N, epi=0,
         accumulate=1, variant=variant)
    want = round_bf16((c0 + round_bf16(v).astype(np.float64)).astype(np.float32))
    got = Cd.float().cpu().numpy()
    assert np.array_equal(got, want), int((got != want).sum())


@pytest.mark.parametrize("n", [1, 7, 4096, (1 << 20) + 3])
def test_adamw_bit_exact_vs_oracle(lib, n):
    """K9 vs oracle AdamW (fp32, D-14 op order): bit-identical theta, m, v, theta16."""
    t = torch()
    from oracle import adamw
    from synth import adam_test_state
    theta, m, v, g = adam_test_state(n, seed=n)
    sc = adamw.step_scalars(3)
    scal = np.array([sc[k] for k in ("decay", "b1", "omb1", "b2", "omb2", "step", "bc2_sqrt",
                                     "eps", "inv_scale")], dtype=np.float32)
    dth = t.from_numpy(theta.copy()).cuda()
    dm = t.from_numpy(m.copy()).cuda()
    dv = t.from_numpy(v.copy()).cuda()
    dg = t.from_numpy(g).to(t.bfloat16).cuda()
    d16 = t.empty(n, dtype=t.bfloat16, device="cuda")
    rc = lib.axonn_k_adamw(n, dg.data_ptr(), dth.data_ptr(), dm.data_ptr(), dv.data_ptr(),
                           d16.data_ptr(), scal.ctypes.data_as(C.POINTER(C.c_float)), None)
    assert rc == 0
    t.cuda.synchronize()
    th_r, m_r, v_r = theta.copy(), m.copy(), v.copy()
    t16 = adamw.adamw_step_fp32(th_r, m_r, v_r, g, sc)
    assert np.array_equal(dth.cpu().numpy().view(np.uint32), th_r.view(np.uint32))
    assert np.array_equal(dm.cpu().numpy().view(np.uint32), m_r.view(np.uint32))
    assert np.array_equal(dv.cpu().numpy().view(np.uint32), v_r.view(np.uint32))
    assert np.array_equal(d16.float().cpu().numpy().view(np.uint32), t16.view(np.uint32))


@pytest.mark.parametrize("M,N,K,epi", [(1024, 1536, 1024, 1), (1000, 1000, 1000, 0), (1024, 1536, 1024, 2),
                                       (4096, 2048, 2048, 0), (2048, 2048, 4096, 3), (256, 256, 1024, 0),
                                       (256, 256, 1024, 3)])
def test_gemm_ragged_waves_and_epilogues(lib, M, N, K, epi):
    """Shapes whose tile count is not a multiple of the 74 CTA pairs (ragged last wave) and
    whose M / N / K are not tile multiples, through every linear-layer epilogue: values vs the
    definition, and bitwise run-to-run."""
    t = torch()
    A = dev_bf16(RNG.standard_normal((M, K)) * 0.5)
    B = dev_bf16(RNG.standard_normal((N, K)) * 0.05)
    bias = dev_bf16(RNG.standard_normal(N) * 0.1)
    aux = dev_bf16(RNG.standard_normal((M, N)))
    outs = []
    for _ in range(2):
        if epi == 3:
            Cd = t.zeros((M, N), dtype=t.float32, device="cuda")
            gemm(lib, M=M, N=N, K=K, A=A, lda=K, B=B, ldb=K, C=Cd, ldc=N, epi=3, accumulate=1)
        elif epi == 1:
            Cd = t.empty((M, N), dtype=t.bfloat16, device="cuda")
            pre = t.empty((M, N), dtype=t.bfloat16, device="cuda")
            gemm(lib, M=M, N=N, K=K, A=A, lda=K, B=B, ldb=K, C=Cd, ldc=N, epi=1, bias=bias, aux=pre, ld_aux=N)
        elif epi == 2:
            Cd = t.empty((M, N), dtype=t.bfloat16, device="cuda")
            gemm(lib, M=M, N=N, K=K, A=A, lda=K, B=B, ldb=K, C=Cd, ldc=N, epi=2, aux=aux, ld_aux=N)
        else:
            Cd = t.empty((M, N), dtype=t.bfloat16, device="cuda")
            gemm(lib, M=M, N=N, K=K, A=A, lda=K, B=B, ldb=K, C=Cd, ldc=N, epi=0, bias=bias, resid=aux,
                 ld_resid=N)
        outs.append(Cd.clone())
    assert t.equal(outs[0], outs[1])
    acc = host(A) @ host(B).T
    c = 0.7978845608028654
    if epi == 3:
        ref = acc
    elif epi == 1:
        p = acc + host(bias)
        ref = 0.5 * p * (1 + np.tanh(c * (p + 0.044715 * p ** 3)))
    elif epi == 2:
        a = host(aux)
        th = np.tanh(c * (a + 0.044715 * a ** 3))
        ref = acc * (0.5 * (1 + th) + 0.5 * a * (1 - th * th) * c * (1 + 3 * 0.044715 * a * a))
    else:
        ref = acc + host(bias) + host(aux)
    out = outs[0].float().cpu().numpy().astype(np.float64)
    assert rel(out, ref) < (1e-5 if epi == 3 else 1e-2)


def test_calibrate_speed_is_plausible(lib):
    """axonn_calibrate_speed (reading D-21c) on the 1.3B FC1 shape: K1's sustained TFLOP/s
    lies between half the bf16 peak and the nominal 2.25 PFLOP/s, and the call leaves the
    device usable (a second call agrees within 25 %)."""
    a, b = C.c_double(), C.c_double()
    assert lib.axonn_calibrate_speed(0, 4096, 8192, 2048, 200, C.byref(a)) == 0
    assert lib.axonn_calibrate_speed(0, 4096, 8192, 2048, 200, C.byref(b)) == 0
    assert 700.0 < a.value < 2250.0 and 700.0 < b.value < 2250.0, (a.value, b.value)
    assert abs(a.value - b.value) <= 0.25 * max(a.value, b.value)
