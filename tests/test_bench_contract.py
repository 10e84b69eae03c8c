"""bench.py output contract on CPU: `--impl reference` (the oracle arm, ④) prints exactly one
JSON line on stdout with the keys the driver reads; everything else goes to stderr."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "tiny", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_reports_the_steps_it_ran():
    """The reference line's steps x ms_per_step is its measured timed wall time (every step is
    one oracle sample; nothing is extrapolated or skipped)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "tiny", "--steps", "3", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["steps"] == 3 and d["warmup"] == 1
    assert abs(d["steps"] * d["ms_per_step"] / 1e3 - d["timed_wall_s"]) <= 1e-6 * d["timed_wall_s"] + 1e-9


def test_default_workload_per_gpu_count(monkeypatch):
    """--config auto: gpt1.3b (configs[1]) at N = 1; the north-star 12B grid (configs[2]) at
    N >= 2: 2 x 1 (24 layers), 4 x 1 (48), 4 x 2 (48) at N = 2, 4, 8 -- 12 layers per stage."""
    sys.path.insert(0, ROOT)
    import bench
    want = {1: ("gpt1.3b", 1, 24, 1), 2: ("gpt12b", 2, 24, 1), 4: ("gpt12b", 4, 48, 1),
            8: ("gpt12b", 4, 48, 2)}
    for n, (name, gi, layers, gd) in want.items():
        monkeypatch.setenv("WORLD_SIZE", str(n))
        args, cfg = bench.parse_args([])
        assert (args.config, cfg["g_inter"], cfg["n_layers"], n // cfg["g_inter"]) == (name, gi, layers, gd)
        if name == "gpt12b":
            assert cfg["hidden"] == 4512 and cfg["heads"] == 24 and cfg["microbatch"] == 8
            assert cfg["mb_per_replica"] == 64


def test_memory_ledger_half_accumulation():
    """The bench line's `memory`: the paper's 20 phi / 4 phi +
    16 bsize beside ours, 2 phi theta16 + 2 phi half grad + 4 phi32 fp32 accumulators + (12 phi
    | 36 bsize ring); with grad_accum_fp32 = 0 (D-38) phi32 counts only the vectors and the
    embedding tables."""
    sys.path.insert(0, ROOT)
    import bench

    class Oc:
        def __init__(self, fp32):
            self.bucket_elems, self.grad_accum_fp32 = 1000, fp32

    class Eng:
        def __init__(self, fp32):
            self.oc = Oc(fp32)

        def tensors(self):
            return [("tok_emb", (10, 4), 40), ("l0.ln1_g", (4,), 4), ("l0.w_qkv", (12, 4), 48),
                    ("l0.b_qkv", (12,), 12), ("l0.w_fc2", (4, 16), 64), ("head_w", (10, 4), 40)]

    phi = 40 + 4 + 48 + 12 + 64 + 40
    full = bench.memory_ledger(Eng(1), offload=False)
    assert full["phi_fp32_accum"] == phi
    assert full["ours_model_state_bytes"] == 4 * phi + 4 * phi + 12 * phi == full["paper_model_state_bytes"]
    half = bench.memory_ledger(Eng(0), offload=True)
    phi32 = 40 + 4 + 12
    assert half["phi_fp32_accum"] == phi32
    assert half["ours_model_state_bytes"] == 4 * phi + 4 * phi32 + 36 * 1000
    assert half["paper_model_state_bytes"] == 4 * phi + 16 * 1000
