"""bench.py — AxoNN hybrid training step on B200 (BASELINE.json metric).

One step = one AxoNN batch: axonn_run_batch (Alg. 1 l.4-6: Alg. 2 inter-layer
step of every microbatch, fp32 weight-gradient accumulation, bf16 gradient
all-reduce over the column) + axonn_optimizer_step (AdamW over every
parameter, bucketed, overlapped with the all-reduce chunks).  Nothing is
skipped inside the timed region.

Default workload (`--config auto`):
* N = 1: BASELINE.json configs[1], the GPT 1.3B-shaped model (24 layers, hidden 2048,
  16 heads, seq 512, vocab 51200), G_inter = 1, microbatch 32, 2 microbatches (64 samples),
  optimizer state in HBM.  At G_inter = 1 the microbatch size only trades activation memory
  for GEMM size (b_m 8 / 16 / 32 / 64: 967-973 / 1015 / 1042 / 1053 TFLOP/s, 34 / 41 / 54 / 81
  GiB; profiles/r1/bench_1p3b_mb_sweep_r56.log).
* N >= 2: the north-star target, BASELINE.json configs[2]: the paper's 12B transformer shape
  (Table I: h 4512, 24 heads) on the grid G_inter = min(4, N) x G_data =
  N / G_inter with 12 layers per stage (4 x 2 at N = 8 is the 48-layer 12B model; 4 x 1 at
  N = 4 the same stages without the second replica; 2 x 1 at N = 2 the SURVEY's 24-layer
  2-GPU proxy), microbatch 8 (Table II), 64 microbatches per replica, bsize 4M,
  k 4.  Offload off by default (the 12-layer stage fits in 180 GB);
  `--offload 1` selects the bucketed pinned-host optimizer.  Weak scaling: per-GPU work is
  one 12-layer stage of 64 microbatches at every N.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun every rank runs one GPU; rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")   # before any CUDA context

_JSON_FD = 1   # main() points fd 1 at stderr and keeps the real stdout here


def emit(out: dict) -> None:
    """Write the one JSON line to the real stdout (NCCL's native banner and any other
    native prints land on stderr)."""
    os.write(_JSON_FD, (json.dumps(out) + "\n").encode())


METRIC = "per-GPU model TFLOP/s and % of B200 bf16 peak at 1/2/4/8 GPUs; batch time"

CONFIGS = {
    # BASELINE.json configs[2]: the 12B transformer shape on the G_inter = min(4, N) x
    # G_data = N / G_inter grid, 12 layers per stage (the 48-layer model at G_inter = 4)
    "gpt12b": dict(layers_per_stage=12, hidden=4512, heads=24, seq_len=512, vocab=51200,
                   g_inter="grid", microbatch=8, mb_per_replica=64, offload=False),
    # BASELINE.json configs[1]: GPT 1.3B-shaped, G_inter = 1, G_data = N, no offload
    "gpt1.3b": dict(n_layers=24, hidden=2048, heads=16, seq_len=512, vocab=51200,
                    g_inter=1, microbatch=32, mb_per_replica=2, offload=False),
    # small smoke configuration (BASELINE.json configs[0] shape, single stage)
    "tiny": dict(n_layers=2, hidden=64, heads=2, seq_len=32, vocab=256,
                 g_inter=1, microbatch=2, mb_per_replica=4, offload=False),
    # BASELINE.json configs[2] proxy: the paper's 12B layer shape (Table I),
    # 12 layers per stage as in the 4 x 2 grid, G_inter = N (pipeline), microbatch 8, m = 64 per replica
    # (Table II), bucketed CPU-offloaded Adam (bsize 4M, k 4)
    "gpt12b-pipe": dict(layers_per_stage=12, hidden=4512, heads=24, seq_len=512, vocab=51200,
                        g_inter="N", microbatch=8, mb_per_replica=64, offload=True),
    # BASELINE.json configs[3] proxy: the 24B layer shape (d = 176), 6 layers per stage as in
    # 8 x 1, microbatch 4, offload on
    "gpt24b-pipe": dict(layers_per_stage=6, hidden=6336, heads=36, seq_len=512, vocab=51200,
                        g_inter="N", microbatch=4, mb_per_replica=32, offload=True),
}


def memory_ledger(eng, offload):
    """Model-state bytes of rank 0's stage: the paper's
    ledger, 20 phi without offload and 4 phi + 16 bsize with it, beside this build's:
    theta16 2 phi + half gradient 2 phi + fp32 gradient accumulators (4 phi, reading D-20; with
    grad_accum_fp32 = 0 only the vectors and embedding tables, 4 phi32, reading D-38), plus
    theta32 / m / v (12 phi) in HBM or a 3-slot device ring of 36 bsize (D-34) with 12 phi in
    pinned host memory.  Activations come on top."""
    mats = ("w_qkv", "w_o", "w_fc1", "w_fc2", "head_w")
    phi = sum(n for _, _, n in eng.tensors())
    phi32 = phi if eng.oc.grad_accum_fp32 else \
        sum(n for name, _, n in eng.tensors() if name.split(".")[-1] not in mats)
    bsize = eng.oc.bucket_elems
    ours = 4 * phi + 4 * phi32 + (36 * bsize if offload else 12 * phi)
    return {"phi_stage": phi, "phi_fp32_accum": phi32, "bsize": bsize,
            "paper_model_state_bytes": 4 * phi + 16 * bsize if offload else 20 * phi,
            "ours_model_state_bytes": ours, "host_pinned_bytes": 12 * phi if offload else 0,
            "note": "rank 0's stage; ours = 2phi theta16 + 2phi half grad + 4phi32 fp32 grad "
                    "accumulators (D-20 / D-38) + (36 bsize ring | 12 phi theta32/m/v); "
                    "device_mem_gib adds activations"}


def model_flops(b, s, l, h, V):
    """72 b s l h^2 (1 + s/6h) + 6 b s h V (reading D-25; Eq. 3 credits recompute)."""
    return 72 * b * s * l * h * h + 12 * b * s * s * l * h + 6 * b * s * h * V


def eq3_flops(b, s, l, h, V):
    return 96 * b * s * l * h * h + 16 * b * s * s * l * h + 6 * b * s * h * V


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=d.get("hbm_gbs", 6456.2), bf16=d.get("bf16_tflops", 1660.9),
                    bf16_sus=d.get("bf16_tflops_sustained", 1415.3), src="MEASURED_PEAKS.json")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="B200_PROFILING.md fallback")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def k1_traffic(cfg):
    """roofline.traffic: DRAM bytes per K1 launch from the committed `ncu --set full` capture of
    one layer's linear-layer GEMMs (profiles/r1/k1_traffic.json, scripts/ncu_traffic.py), beside
    the algorithmic bytes per launch of the same launches (operands read once, outputs written
    once).  null when no capture matches this model width and microbatch."""
    p = None
    for rnd in ("r2", "r1"):   # the latest round's capture
        cand = os.path.join(ROOT, "profiles", rnd, "k1_traffic.json")
        if os.path.exists(cand):
            p = cand
            break
    if p is None:
        return {"traffic": None}
    d = json.load(open(p))
    if d.get("hidden") != cfg["hidden"] or d.get("tokens") != cfg["microbatch"] * cfg["seq_len"]:
        return {"traffic": None}
    # the capture is one 1-layer microbatch (12 layer GEMMs + 3 LM-head GEMMs); `achieved`
    # averages over the K1 launches of one n_layers microbatch, so weight the layer launches
    # by n_layers to average over the same population
    ls = d.get("launches", [])
    if ls and all("gemm" in l and "algorithmic_bytes" in l for l in ls):
        L = cfg["n_layers"]
        w = [1 if "head" in l["gemm"] else L for l in ls]
        n = sum(w)
        dram = sum(wi * l["dram_total"] for wi, l in zip(w, ls)) / n
        alg = sum(wi * l["algorithmic_bytes"] for wi, l in zip(w, ls)) / n
        unit = f"bytes per K1 launch (average over one microbatch: {L} x 12 layer GEMMs + 3 head)"
    else:
        dram, alg = d["dram_bytes_per_launch_avg"], d.get("algorithmic_bytes_per_launch_avg")
        unit = "bytes per K1 launch (average over the captured launches)"
    return {"traffic": dram, "traffic_algorithmic": alg, "traffic_unit": unit,
            "traffic_src": os.path.relpath(p, ROOT) + " (ncu --set full, 1-layer microbatch)"}


def _blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [d.get("num_threads", 0) for d in threadpool_info() if d.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:   # pragma: no cover
        return os.cpu_count() or 1


def oracle_layer_sample(cfg, steps: int = 1):
    """One timed oracle sample of the configured workload: one transformer layer of the
    configured shape as a middle pipeline stage (nn_shard.Forward + Backward, no embedding /
    head) on one full-length sequence, fp64 numpy on the host cores.  Returns (seconds per
    sample, model FLOPs of the sample = 72 s h^2 (1 + s/6h), description)."""
    from oracle import model as om
    from synth import init_params
    c = om.GPTConfig(n_layers=3, hidden=cfg["hidden"], heads=cfg["heads"], seq_len=cfg["seq_len"],
                     vocab=cfg["vocab"])
    names = om.layer_names(1)
    rng = np.random.default_rng(5)
    full = init_params(1, c.hidden, c.seq_len, 8, seed=5, parity=False)
    p = {n.replace("l0.", "l1."): v.astype(np.float64) for n, v in full.items() if n.startswith("l0.")}
    assert set(p) == set(names)
    x = rng.standard_normal((1, c.seq_len, c.hidden))
    dy = rng.standard_normal((1, c.seq_len, c.hidden)) * 1e-3
    t0 = time.perf_counter()
    for _ in range(steps):
        out, cache = om.stage_forward(p, c, 1, 3, x)
        om.stage_backward(p, c, 1, 3, cache, dy)
    dt = (time.perf_counter() - t0) / steps
    fl = 72 * c.seq_len * c.hidden ** 2 + 12 * c.seq_len ** 2 * c.hidden
    desc = (f"numpy fp64 oracle nn_shard Forward+Backward of one layer (h {c.hidden}, a {c.heads}, "
            f"s {c.seq_len}) on 1 x {c.seq_len} tokens")
    return dt, fl, desc


def cpu_baseline(cfg, batch_flops: float):
    """the oracle as it stands, timed on the host cores (never the target).
    value = item 2, the oracle's model TFLOP/s on one layer of the configured shape; beside it
    the EXTRAPOLATED oracle time of the whole configured batch (model FLOPs / that rate), item 3
    (oracle AdamW over 2^26 parameters, GB/s at 28 B/param) and item 1 (the full tiny step:
    Alg. 1 + Alg. 2 over 2 x 1 virtual workers, 4 microbatches, plus its AdamW).  About 10-30 s."""
    from oracle import adamw as oa
    from oracle import hybrid as oh
    from oracle import model as om
    from synth import init_params, markov_tokens
    dt, fl, desc = oracle_layer_sample(cfg, 1)
    rate = fl / dt
    # item 3: AdamW over 2^26 fp32 parameters (in place), bf16 gradients
    n = 1 << 26
    rng = np.random.default_rng(3)
    th = (rng.standard_normal(n) * 0.02).astype(np.float32)
    mm = np.zeros(n, np.float32)
    vv = np.zeros(n, np.float32)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    t0 = time.perf_counter()
    oa.adamw_step_fp32(th, mm, vv, g, oa.step_scalars(1))
    t_adam = time.perf_counter() - t0
    del th, mm, vv, g
    # item 1: the full tiny step (BASELINE.json configs[0]) on 2 x 1 virtual workers
    tc = om.GPTConfig(n_layers=2, hidden=64, heads=2, seq_len=32, vocab=256)
    tp = {k: v.astype(np.float64) for k, v in init_params(2, 64, 32, 256, seed=42).items()}
    tok = markov_tokens(8, 32, 256, seed=7)
    t0 = time.perf_counter()
    _, tg = oh.hybrid_step(tp, tc, tok, 2, 1, 2)
    sc = oa.step_scalars(1)
    for k, v in tp.items():
        t32 = v.astype(np.float32)
        oa.adamw_step_fp32(t32, np.zeros_like(t32), np.zeros_like(t32), tg[k].astype(np.float32), sc)
    t_tiny = time.perf_counter() - t0
    return dict(value=rate / 1e12, unit="model TFLOP/s", cores=_blas_threads(), kind="oracle",
                sample=f"{desc}, {dt:.2f} s/sample",
                extrapolated_batch_s=batch_flops / rate,
                adamw_gbs=28.0 * n / t_adam / 1e9, adamw_params=n,
                tiny_step_s=t_tiny, host_cpus=os.cpu_count())


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle (this tier's reference arm) on the host, rank 0 only.
    Every step is one bounded oracle sample of the configured workload (oracle_layer_sample);
    W untimed + K timed samples, so steps x ms_per_step is the timed wall time."""
    if rank != 0:
        return
    for _ in range(args.warmup):
        oracle_layer_sample(cfg, 1)
    t0 = time.perf_counter()
    dts = []
    for _ in range(args.steps):
        dt, fl, desc = oracle_layer_sample(cfg, 1)
        dts.append(dt)
    wall = time.perf_counter() - t0
    ms = wall * 1e3 / max(args.steps, 1)
    v = fl / (ms / 1e3) / 1e12
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "model TFLOP/s (all GPUs)",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "timed_wall_s": wall,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": {"workload": args.config, "global_batch": 1, "seq_len": cfg["seq_len"],
                      "parallelism": "cpu oracle", "sample": desc},
           "cpu_baseline": {"value": v, "unit": "model TFLOP/s", "cores": _blas_threads(),
                            "kind": "oracle", "sample": f"{desc}, one sample per step"},
           "e2e": {"value": v, "unit": "model TFLOP/s (all GPUs)", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    emit(out)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="auto", choices=["auto"] + sorted(CONFIGS),
                    help="auto: gpt1.3b at N = 1, gpt12b (G_inter = min(4, N) grid) at N >= 2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--layers", type=int, default=None, help="override n_layers (profiling runs only)")
    ap.add_argument("--mb-per-replica", type=int, default=None, help="microbatches per replica (m)")
    ap.add_argument("--microbatch", type=int, default=None, help="microbatch size b_m (rows)")
    ap.add_argument("--offload", type=int, default=None, help="1/0: override the config's offload")
    ap.add_argument("--checkpoint-interval", type=int, default=0,
                    help="activation checkpointing ac (PAPER.md:553-576): 0 off, -1 the paper's rule")
    ap.add_argument("--overlap-next-batch", type=int, default=None,
                    help="1/0: optimizer step t overlaps batch t+1 (default: on with offload only)")
    ap.add_argument("--pipeline-limit", type=int, default=0,
                    help="microbatches in flight per pipeline (0: G_inter, PAPER.md:467-470)")
    ap.add_argument("--stage-balance", type=int, default=None,
                    help="1: half-layer stage boundaries balancing the LM head (reading D-21b); "
                         "2: the same, weighted by each stage's measured GPU speed (D-21c); "
                         "default on unless activation checkpointing is requested")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp16"],
                    help="half format (library build); fp16 runs with a static loss scale (D-11)")
    ap.add_argument("--loss-scale", type=float, default=None,
                    help="static loss scale S (default 1 for bf16, 1024 for fp16)")
    ap.add_argument("--g-inter", type=int, default=None,
                    help="pipeline stages (pipeline configs; G_data = N / G_inter)")
    ap.add_argument("--coarsen-k", type=int, default=4,
                    help="all-reduce chunk = k * bsize elements (PAPER.md:731-737; paper 4)")
    ap.add_argument("--bucket-elems", type=int, default=4_000_000,
                    help="optimizer bucket bsize in elements (PAPER.md:683; paper 4M)")
    ap.add_argument("--grad-accum-fp32", type=int, default=1,
                    help="0: the paper's footprint, weight matrices accumulate in the half "
                         "gradient (reading D-38)")
    args = ap.parse_args(argv)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.stage_balance is None:
        args.stage_balance = int(args.checkpoint_interval in (0, 1))
    args.config, cfg = resolve_config(args, world_env)
    return args, cfg


def resolve_config(args, world: int):
    """(workload name, config dict) the run measures: --config auto picks gpt1.3b at N = 1 and
    the north-star 12B grid (G_inter = min(4, N) x G_data = N / G_inter) at N >= 2."""
    name = args.config
    if name == "auto":
        name = "gpt1.3b" if world == 1 else "gpt12b"
    cfg = dict(CONFIGS[name])
    if args.layers:
        cfg["n_layers"] = args.layers
    if args.mb_per_replica:
        cfg["mb_per_replica"] = args.mb_per_replica
    if args.microbatch:
        cfg["microbatch"] = args.microbatch
    if args.offload is not None:
        cfg["offload"] = bool(args.offload)
    if cfg.get("g_inter") == "N":   # pipeline proxies: one stage per GPU unless --g-inter
        cfg["g_inter"] = args.g_inter or world
        cfg.setdefault("n_layers", cfg["layers_per_stage"] * cfg["g_inter"])
    elif cfg.get("g_inter") == "grid":   # north-star grid: G_inter = min(4, N)
        cfg["g_inter"] = args.g_inter or min(4, world)
        cfg.setdefault("n_layers", cfg["layers_per_stage"] * cfg["g_inter"])
    return name, cfg


def main(argv=None):
    args, cfg = parse_args(argv)
    from paper_2110_13005_b200 import dist as D
    rank, world, local = D.env_rank_world()
    if world == 1 and args.gpus > 1:
        raise SystemExit("use torchrun --nproc-per-node N for N > 1")
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    torch.cuda.set_device(local)
    D.init_process_group(rank, world, backend="gloo")
    from paper_2110_13005_b200.engine import AxoNN
    g_inter = cfg["g_inter"]
    g_data = world // g_inter
    b_m, m = cfg["microbatch"], cfg["mb_per_replica"]
    B = b_m * m * g_data
    nid = D.share_unique_id(rank, world, D.nccl_unique_id)
    eng = AxoNN(g_inter, g_data, b_m, n_layers=cfg["n_layers"], hidden=cfg["hidden"],
                heads=cfg["heads"], seq_len=cfg["seq_len"], vocab=cfg["vocab"], init_seed=42,
                offload=cfg["offload"], rank=rank, world_size=world, device=local, nccl_id=nid,
                checkpoint_interval=args.checkpoint_interval, dtype=args.dtype,
                stage_balance="calibrate" if args.stage_balance == 2 else bool(args.stage_balance),
                pipeline_limit=args.pipeline_limit, coarsen_k=args.coarsen_k,
                bucket_elems=args.bucket_elems, grad_accum_fp32=bool(args.grad_accum_fp32),
                overlap_next_batch=None if args.overlap_next_batch is None else bool(args.overlap_next_batch),
                loss_scale=args.loss_scale or (1024.0 if args.dtype == "fp16" else 1.0))
    from synth import uniform_tokens
    s, V = cfg["seq_len"], cfg["vocab"]
    tokens = uniform_tokens(B, s, V, seed=1234)          # full batch on the host (pinned below)
    j = rank // g_inter
    lo, hi = D.batch_shard(B, g_data, j)
    d_tok = torch.from_numpy(tokens[lo:hi].copy()).cuda()  # this replica's shard resident in HBM
    h_tok = torch.from_numpy(tokens).pin_memory()
    h_np = h_tok.numpy()

    # warm-up (untimed)
    for _ in range(args.warmup):
        eng.run_batch_device(d_tok.data_ptr(), B)
        eng.optimizer_step()
    torch.cuda.synchronize()

    # timed region: K plain steps with device-resident inputs (no instrumentation)
    ph = {"t_pipe_ms": 0.0, "t_busy_ms": 0.0, "t_allreduce_ms": 0.0, "t_opt_exposed_ms": 0.0}
    launches = 0
    D.barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        eng.timer_mark(0)
        losses = []
        for step in range(args.steps):
            losses.append(eng.run_batch_device(d_tok.data_ptr(), B))
            eng.optimizer_step()
            st = eng.stats()
            launches += int(st["kernel_launches"])
            for k in ph:
                ph[k] += st[k] / args.steps
        eng.timer_mark(1)
        dev_ms = eng.timer_elapsed_ms(0, 1)
    torch.cuda.synchronize()
    D.barrier(world)
    dev_ms = D.max_over_ranks(dev_ms, world)
    bubble = 1.0 - ph["t_busy_ms"] / ph["t_pipe_ms"] if ph["t_pipe_ms"] > 0 else 0.0
    bubble_ranks = D.gather_to_all(bubble, world)   # every rank joins the collective
    bubble_max = max(bubble_ranks)
    ms_step = dev_ms / args.steps
    fl = model_flops(B, s, cfg["n_layers"], cfg["hidden"], V)
    value = fl / (ms_step / 1e3) / 1e12                       # whole-job model TFLOP/s

    # one extra, instrumented step AFTER the timed region: the K1 / K2 launches of its middle
    # microbatch ((m - 1) / 2, clear of the optimizer chunks of the last backward) and its K9
    # launches are bracketed by CUDA events on their launching streams
    # (roofline and per-shape numbers; the profiled microbatch runs its weight gradients in
    # order on the compute stream so each event pair times one launch)
    overlap = cfg["offload"] if args.overlap_next_batch is None else bool(args.overlap_next_batch)
    eng.set_profiling(True)
    nvtx = os.environ.get("AXONN_NVTX") == "1"   # ncu --nvtx-include profiled_step/
    if nvtx:
        torch.cuda.nvtx.range_push("profiled_step")
    eng.run_batch_device(d_tok.data_ptr(), B)
    eng.optimizer_step()
    if nvtx:
        torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    st = eng.stats()
    gemm_ms, gemm_flop = st["gemm_ms"], st["gemm_flop"]
    adam_ms, adam_bytes = st["adam_ms"], st["adam_bytes"]
    breakdown = {k: list(v) for k, v in eng.profile().items()}
    eng.set_profiling(False)
    if overlap:   # the overlapped optimizer's records complete during the next batch
        eng.run_batch_device(d_tok.data_ptr(), B)
        eng.optimizer_step()
        st2 = eng.stats()
        adam_ms, adam_bytes = st2["adam_ms"], st2["adam_bytes"]
        for k, v in eng.profile().items():
            if k == "adamw":
                breakdown[k] = list(v)

    # e2e: through the public C-ABI with HOST tokens; H2D of the shard + D2H of
    # the loss happen inside axonn_run_batch every step
    e2e_steps = args.e2e_steps or max(1, min(args.steps, 3))
    D.barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        eng.run_batch(h_np)
        eng.optimizer_step()
    torch.cuda.synchronize()
    e2e_ms = D.max_over_ranks((time.perf_counter() - t0) * 1e3 / e2e_steps, world)
    e2e_val = fl / (e2e_ms / 1e3) / 1e12

    peaks = load_peaks()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:   # the CPU baseline is an N = 1 figure
        cpu = cpu_baseline(cfg, fl)
    if rank == 0:
        gemm_tf = gemm_flop / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
        out = {
            "metric": METRIC,
            "value": value,
            "unit": "model TFLOP/s (all GPUs)",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": args.dtype,
            "data": "synthetic (uniform tokens, splitmix64 seed 1234; random-init weights seed 42)",
            "config": {"workload": args.config, "model": f"GPT {cfg['n_layers']}L h{cfg['hidden']} "
                       f"a{cfg['heads']} s{s} V{V}", "global_batch": B, "seq_len": s,
                       "microbatch": b_m, "microbatches_per_replica": m,
                       "parallelism": f"G_inter{g_inter} x G_data{g_data}",
                       "offload": cfg["offload"], "checkpoint_interval": args.checkpoint_interval,
                       "grad_accum_fp32": args.grad_accum_fp32,
                       "stage_balance": args.stage_balance, "pipeline_limit": args.pipeline_limit,
                       "stage_blocks": eng.partition() if args.stage_balance else None,
                       "stage_speed_tflops": eng.stage_speed,
                       "l2": "inputs larger than L2 (GBs of weights/activations per step)"},
            "per_gpu_tflops": value / world,
            "device_mem_gib": torch.cuda.mem_get_info()[1] / 2**30 - torch.cuda.mem_get_info()[0] / 2**30,
            "memory": memory_ledger(eng, cfg["offload"]),
            "pct_bf16_peak": 100.0 * value / world / peaks["bf16"],
            "pct_bf16_peak_sustained": 100.0 * value / world / peaks["bf16_sus"],
            "eq3_tflops_per_gpu": eq3_flops(B, s, cfg["n_layers"], cfg["hidden"], V) / (ms_step / 1e3) / 1e12 / world,
            "batch_time_s": ms_step / 1e3,
            "loss": losses[-1] if losses else None,
            # device-timed phases per step (CUDA events, rank 0; PAPER.md:704-708 phase bars):
            # Alg. 2 phase, this stage's Forward/Backward busy time in it, the gradient cast +
            # column all-reduce after it, optimizer time after the all-reduce
            "phases": {"pipeline_ms": ph["t_pipe_ms"], "compute_busy_ms": ph["t_busy_ms"],
                       "bubble_frac": bubble, "bubble_frac_max_over_ranks": bubble_max,
                       "bubble_frac_per_rank": bubble_ranks,
                       "predicted_bubble_frac": (g_inter - 1) / (m + g_inter - 1),
                       "allreduce_exposed_ms": ph["t_allreduce_ms"],
                       "optimizer_exposed_ms": ph["t_opt_exposed_ms"],
                       "note": "with overlap_next_batch (offload) the optimizer figure is the previous step's"},
            "clocks": clk.summary(),
            "e2e": {"value": e2e_val, "unit": "model TFLOP/s (all GPUs)",
                    "h2d_bytes_per_step": int((hi - lo) * (s + 1) * 4), "d2h_bytes_per_step": 8,
                    "ms_per_step": e2e_ms},
            "gpu_launches": launches,
            "roofline": {"bound": "tensor", "kernel": "K1 gemm_bf16_tcgen05 (linear layers)",
                         "achieved": gemm_tf, "peak": peaks["bf16_sus"], "unit": "TFLOP/s",
                         "frac": (gemm_tf / peaks["bf16_sus"]) if gemm_tf else None,
                         "peak_src": peaks["src"] + " bf16_tflops_sustained (kernel timed inside a long step)",
                         # events bracket the K1 launches of one microbatch (same shapes
                         # each microbatch); share scaled by m
                         "events": "K1 launches of microbatch (m-1)/2 of one instrumented step "
                                   "run after the timed region",
                         "gemm_share_of_step": gemm_ms * m / ms_step,
                         **k1_traffic(cfg)},
            "adam": {"achieved_gbs": adam_bytes / (adam_ms / 1e3) / 1e9 if adam_ms else None,
                     "peak_gbs": peaks["hbm"], "bytes_per_param": 28},
            "cpu_baseline": cpu,
            # per-shape K1 timing (microbatch (m-1)/2 of the instrumented step): ms/launch, TFLOP/s
            "gemm_breakdown": {k: {"ms_per_launch": v[0] / max(v[2], 1),
                                   ("tflops" if k != "adamw" else "GB/s"):
                                       v[1] / (v[0] / 1e3) / (1e12 if k != "adamw" else 1e9)
                                       if v[0] > 0 else None,
                                   "launches": v[2]}
                               for k, v in sorted(breakdown.items(), key=lambda kv: -kv[1][0])},
        }
        emit(out)
    eng.close()


if __name__ == "__main__":
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    main()
