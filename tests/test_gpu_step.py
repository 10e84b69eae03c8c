"""Single-GPU step parity (T3): the CUDA path through the C-ABI vs the oracle.

Same seeded inputs on both sides (synth): bf16-representable weights written
into the library with axonn_write_tensor, Markov tokens (D-23).  Bars from
BASELINE.json north_star: loss rel <= 2e-2 every step, per-tensor gradient
cosine >= 0.999, Adam update bit-identical (<= 1e-6 rel required)."""
import numpy as np
import pytest

from oracle import adamw, model
from oracle.bf16 import round_bf16
from parity import assert_grads_close
from synth import init_params, markov_tokens

pytestmark = pytest.mark.gpu

TINY = dict(n_layers=2, hidden=64, heads=2, seq_len=32, vocab=256)
MINI = dict(n_layers=4, hidden=256, heads=4, seq_len=128, vocab=1024)


def make(cfg, g_inter=1, g_data=1, mb=2, **kw):
    from paper_2110_13005_b200.engine import AxoNN
    return AxoNN(g_inter, g_data, mb, **cfg, **kw)


def cos(a, b):
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    if na < 1e-30 and nb < 1e-30:
        return 1.0
    return float((a * b).sum() / (na * nb))


def oracle_grads(params32, cfg, tokens):
    p = {k: v.astype(np.float64) for k, v in params32.items()}
    c = model.GPTConfig(**cfg)
    return model.full_batch_loss_and_grads(p, c, tokens)


PAD10 = dict(n_layers=2, hidden=80, heads=8, seq_len=32, vocab=256)     # d = 10 -> padded 16
PAD188 = dict(n_layers=1, hidden=376, heads=2, seq_len=64, vocab=512)   # the 12B head dim d = 188


@pytest.mark.parametrize("cfg,B,mb", [(TINY, 8, 2), (TINY, 8, 8), (MINI, 16, 2), (PAD10, 8, 2),
                                      (PAD188, 4, 2)])
def test_step_loss_and_grads_vs_oracle(cfg, B, mb):
    from paper_2110_13005_b200.engine import T_GRAD32, T_MASTER
    eng = make(cfg, mb=mb)
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    eng.write_all(T_MASTER, params)
    tok = markov_tokens(B, cfg["seq_len"], cfg["vocab"], seed=7)
    loss = eng.run_batch(tok)
    loss_ref, g_ref = oracle_grads(params, cfg, tok)
    assert abs(loss - loss_ref) <= 2e-2 * abs(loss_ref), (loss, loss_ref)
    g = eng.read_all(T_GRAD32)
    assert_grads_close(g, g_ref, where=f"{cfg} B {B} mb {mb}")
    eng.close()


def test_optimizer_step_bit_exact_and_theta16():
    """Isolated AdamW inside the engine: the GPU update of (theta32, m, v) from
    the GPU's own bf16 gradients equals the oracle's fp32 AdamW bitwise, and
    theta16 == RNE(theta32)."""
    from paper_2110_13005_b200.engine import T_ADAM_M, T_ADAM_V, T_GRAD, T_MASTER, T_PARAM16
    cfg = TINY
    eng = make(cfg, bucket_elems=1000, coarsen_k=2)
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    eng.write_all(T_MASTER, params)
    tok = markov_tokens(8, cfg["seq_len"], cfg["vocab"], seed=7)
    for step in (1, 2, 3):
        eng.run_batch(tok)
        g16 = eng.read_all(T_GRAD)
        th, m, v = eng.read_all(T_MASTER), eng.read_all(T_ADAM_M), eng.read_all(T_ADAM_V)
        eng.optimizer_step()
        sc = adamw.step_scalars(step)
        for k in th:
            t_r, m_r, v_r = th[k].copy(), m[k].copy(), v[k].copy()
            t16 = adamw.adamw_step_fp32(t_r, m_r, v_r, g16[k], sc)
            got_t = eng.read(T_MASTER, [n for n, _, _ in eng.tensors()].index(k))
            assert np.array_equal(got_t.view(np.uint32), t_r.view(np.uint32)), (step, k)
        after = eng.read_all(T_MASTER)
        p16 = eng.read_all(T_PARAM16)
        for k in after:
            assert np.array_equal(p16[k].view(np.uint32), round_bf16(after[k]).view(np.uint32))
        am, av = eng.read_all(T_ADAM_M), eng.read_all(T_ADAM_V)
        for k in am:
            assert np.all(np.isfinite(am[k])) and np.all(av[k] >= 0)
    eng.close()


def test_three_step_training_vs_oracle():
    """Loss trajectory over 3 steps (run_batch + optimizer_step) vs the oracle
    trajectory (fp64 model at theta16, bf16 gradients, fp32 AdamW)."""
    from paper_2110_13005_b200.engine import T_MASTER
    cfg = TINY
    eng = make(cfg)
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    eng.write_all(T_MASTER, params)
    toks = [markov_tokens(8, cfg["seq_len"], cfg["vocab"], seed=100 + i) for i in range(3)]
    theta = {k: v.copy() for k, v in params.items()}
    mm = {k: np.zeros_like(v) for k, v in params.items()}
    vv = {k: np.zeros_like(v) for k, v in params.items()}
    for step, tok in enumerate(toks, start=1):
        loss = eng.run_batch(tok)
        eng.optimizer_step()
        p16 = {k: round_bf16(v) for k, v in theta.items()}
        loss_ref, g = oracle_grads(p16, cfg, tok)
        sc = adamw.step_scalars(step)
        for k in theta:
            adamw.adamw_step_fp32(theta[k], mm[k], vv[k], round_bf16(g[k].astype(np.float32)), sc)
        assert abs(loss - loss_ref) <= 2e-2 * abs(loss_ref), (step, loss, loss_ref)
    eng.close()


def test_offload_equals_in_hbm_bitwise():
    """§8(c.4) item 6: bucketed pinned-host offload == in-HBM optimizer, bitwise."""
    from paper_2110_13005_b200.engine import T_ADAM_V, T_MASTER, T_PARAM16
    cfg = TINY
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    tok = markov_tokens(8, cfg["seq_len"], cfg["vocab"], seed=7)
    res = []
    for off in (0, 1):
        eng = make(cfg, offload=bool(off), bucket_elems=3000, coarsen_k=2)
        eng.write_all(T_MASTER, params)
        for _ in range(2):
            eng.run_batch(tok)
            eng.optimizer_step()
        res.append((eng.read_all(T_MASTER), eng.read_all(T_ADAM_V), eng.read_all(T_PARAM16)))
        eng.close()
    for a, b in zip(res[0], res[1]):
        for k in a:
            assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), k


def test_run_to_run_bitwise_reproducible():
    from paper_2110_13005_b200.engine import T_GRAD32, T_MASTER
    cfg = MINI
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=3)
    tok = markov_tokens(16, cfg["seq_len"], cfg["vocab"], seed=9)
    outs = []
    for _ in range(2):
        eng = make(cfg)
        eng.write_all(T_MASTER, params)
        l = eng.run_batch(tok)
        outs.append((l, eng.read_all(T_GRAD32)))
        eng.close()
    assert outs[0][0] == outs[1][0]
    for k in outs[0][1]:
        assert np.array_equal(outs[0][1][k], outs[1][1][k]), k


def test_state_and_validation_errors():
    from paper_2110_13005_b200.engine import AxoNNError
    with pytest.raises(AxoNNError) as e:
        make(dict(TINY, n_layers=3), g_inter=2, g_data=1)
    assert e.value.status in ("GRID_MISMATCH", "NONDIVISIBLE_LAYERS")
    eng = make(TINY)
    with pytest.raises(AxoNNError) as e:
        eng.optimizer_step()
    assert e.value.status == "STATE"
    tok = markov_tokens(6, TINY["seq_len"], TINY["vocab"], seed=1)
    with pytest.raises(AxoNNError) as e:
        eng.run_batch(tok[:5])
    assert e.value.status == "NONDIVISIBLE_BATCH"
    eng.run_batch(tok[:4])
    with pytest.raises(AxoNNError) as e:
        eng.run_batch(tok[:4])
    assert e.value.status == "STATE"
    eng.optimizer_step()
    eng.close()


@pytest.mark.parametrize("offload", [0, 1])
def test_overlapped_optimizer_equals_synchronous_bitwise(offload):
    """Reading D-32: overlapping optimizer step t with batch t+1 (each layer's forward waits
    only for the buckets holding its parameters) changes no value: losses, theta32, v and
    theta16 after 3 steps are bitwise those of the synchronous schedule."""
    from paper_2110_13005_b200.engine import T_ADAM_V, T_MASTER, T_PARAM16
    cfg = MINI
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=11)
    tok = markov_tokens(16, cfg["seq_len"], cfg["vocab"], seed=5)
    res = []
    for ov in (False, True):
        eng = make(cfg, offload=bool(offload), bucket_elems=40000, coarsen_k=2, overlap_next_batch=ov)
        eng.write_all(T_MASTER, params)
        losses = []
        for _ in range(3):
            losses.append(eng.run_batch(tok))
            eng.optimizer_step()
        res.append((losses, eng.read_all(T_MASTER), eng.read_all(T_ADAM_V), eng.read_all(T_PARAM16)))
        eng.close()
    assert res[0][0] == res[1][0], (res[0][0], res[1][0])
    for a, b in zip(res[0][1:], res[1][1:]):
        for k in a:
            assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), k


@pytest.mark.parametrize("n_layers,g_inter", [(4, 1), (16, 1), (24, 1), (9, 1), (12, 2), (14, 2), (16, 4)])
def test_checkpoint_interval_rule_matches_oracle(n_layers, g_inter):
    """N1: with checkpoint_interval = -1 every stage uses the oracle's
    select_checkpoint_interval (the factor of N / G_inter closest to sqrt(N), ties to the
    smaller; (14, 2) is a case where Eq. 1's argmin differs, 7 vs the rule's 1).  G_inter > 1
    runs as loopback stages on this GPU."""
    from oracle.checkpoint import select_checkpoint_interval
    from paper_2110_13005_b200.engine import AxoNN, LocalGroup, run_stages
    cfg = dict(n_layers=n_layers, hidden=64, heads=2, seq_len=32, vocab=256)
    want = select_checkpoint_interval(n_layers, g_inter)
    if g_inter == 1:
        engs, grp = [AxoNN(1, 1, 2, **cfg, checkpoint_interval=-1)], None
    else:
        grp = LocalGroup(g_inter)
        engs = run_stages(lambda i: AxoNN(g_inter, 1, 2, **cfg, checkpoint_interval=-1, rank=i,
                                          world_size=g_inter, device=0, local_group=grp), g_inter)
    try:
        assert [e.checkpoint_interval() for e in engs] == [want] * g_inter
    finally:
        for e in engs:
            e.close()
        if grp is not None:
            grp.free()


def test_activation_checkpointing_vs_oracle():
    """N1 against the oracle (not only against itself): the rule's interval (ac = 2 for 4
    layers) on a non-periodic batch; loss and every gradient within the parity bars."""
    from parity import oracle_mixed
    from synth import mixed_batch
    from paper_2110_13005_b200.engine import T_GRAD32, T_MASTER
    cfg = MINI
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=21)
    distinct = markov_tokens(3, cfg["seq_len"], cfg["vocab"], seed=31)
    tok, counts = mixed_batch(distinct, 16, seed=4)
    eng = make(cfg, checkpoint_interval=-1)
    eng.write_all(T_MASTER, params)
    loss = eng.run_batch(tok)
    g = eng.read_all(T_GRAD32)
    assert eng.checkpoint_interval() == 2
    eng.close()
    loss_ref, g_ref = oracle_mixed(params, cfg, distinct, counts)
    assert abs(loss - loss_ref) <= 2e-2 * abs(loss_ref), (loss, loss_ref)
    assert_grads_close(g, g_ref, where="checkpointing ac=2")


@pytest.mark.parametrize("ac", [2, 4, -1])
def test_activation_checkpointing_is_bitwise_neutral(ac):
    """§8(f) N1: with checkpointing interval ac the backward recomputes each
    segment's forward from its kept input; the recomputation is the same computation, so the
    loss and every gradient equal those without checkpointing bit for bit."""
    from paper_2110_13005_b200.engine import T_GRAD32, T_MASTER
    cfg = MINI
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=21)
    tok = markov_tokens(16, cfg["seq_len"], cfg["vocab"], seed=4)
    outs = []
    for ck in (0, ac):
        eng = make(cfg, checkpoint_interval=ck)
        eng.write_all(T_MASTER, params)
        loss = eng.run_batch(tok)
        outs.append((loss, eng.read_all(T_GRAD32)))
        eng.close()
    assert outs[0][0] == outs[1][0]
    for k in outs[0][1]:
        assert np.array_equal(outs[0][1][k].view(np.uint32), outs[1][1][k].view(np.uint32)), k


@pytest.mark.parametrize("k", [1, 3])
def test_chunked_gradient_handoff_is_bitwise_neutral(monkeypatch, k):
    """A8: the last backward hands the gradients off chunk by chunk (k * bsize
    elements, cast to the half format as each layer becomes final) and the optimizer runs its
    buckets in chunk-completion order, top chunk first, while the backward is still running.
    Against the hand-off after the pipeline (AXONN_AR_OVERLAP=0, ascending buckets): losses,
    theta32, v and theta16 after 3 steps bitwise equal (AdamW is elementwise, D-16/D-17)."""
    from paper_2110_13005_b200.engine import T_ADAM_V, T_MASTER, T_PARAM16
    cfg = MINI
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=13)
    toks = [markov_tokens(16, cfg["seq_len"], cfg["vocab"], seed=60 + i) for i in range(3)]
    res = []
    for ov in ("0", "1"):
        monkeypatch.setenv("AXONN_AR_OVERLAP", ov)
        eng = make(cfg, bucket_elems=50_000, coarsen_k=k, overlap_next_batch=False)
        eng.write_all(T_MASTER, params)
        losses = []
        for tok in toks:
            losses.append(eng.run_batch(tok))
            eng.optimizer_step()
        res.append((losses, eng.read_all(T_MASTER), eng.read_all(T_ADAM_V), eng.read_all(T_PARAM16)))
        eng.close()
    assert res[0][0] == res[1][0]
    for a, b in zip(res[0][1:], res[1][1:]):
        for name in a:
            assert np.array_equal(a[name].view(np.uint32), b[name].view(np.uint32)), name


def test_token_ids_out_of_range_are_rejected():
    """Token ids index embedding rows and logit columns: an id outside [0, vocab) (host path:
    the whole batch is scanned; device path: a check kernel) returns INVALID_ARG before any
    device work and leaves the context usable; vocab 264 is not a multiple of the embedding
    backward's 32-row blocks, so ids in [264, 288) would otherwise reach past dE_tok."""
    import torch

    from paper_2110_13005_b200.engine import AxoNNError
    cfg = dict(TINY, vocab=264)
    eng = make(cfg)
    tok = markov_tokens(8, cfg["seq_len"], cfg["vocab"], seed=3)
    for bad in (264, 287, -1):
        t2 = tok.copy()
        t2[5, 7] = bad
        with pytest.raises(AxoNNError) as e:
            eng.run_batch(t2)
        assert e.value.status == "INVALID_ARG"
        d = torch.from_numpy(t2).cuda()
        with pytest.raises(AxoNNError) as e:
            eng.run_batch_device(d.data_ptr(), 8)
        assert e.value.status == "INVALID_ARG"
    loss = eng.run_batch(tok)       # still usable
    assert np.isfinite(loss)
    eng.optimizer_step()
    eng.close()
