"""Diagnostic: per-tensor differences between the loopback pipeline and the single-stage run
(tests/test_gpu_loopback.py::test_loopback_pipeline_vs_oracle, MINI G_inter 4), plus
run-to-run repeats of each side."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ.setdefault("AXONN_WATCHDOG_S", "120")
from synth import init_params, markov_tokens, mixed_batch  # noqa: E402
from test_gpu_loopback import MINI, pipeline, single  # noqa: E402

cfg, gi, mb, B = MINI, int(sys.argv[1]) if len(sys.argv) > 1 else 4, 2, 16
params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
distinct = markov_tokens(3, cfg["seq_len"], cfg["vocab"], seed=17)
tok, counts = mixed_batch(distinct, B, seed=B + mb)
runs = {"loop1": pipeline(cfg, gi, mb, params, [tok])[1], "loop2": pipeline(cfg, gi, mb, params, [tok])[1],
        "single1": single(cfg, mb, params, [tok])[1], "single2": single(cfg, mb, params, [tok])[1]}
for a, b in (("loop1", "loop2"), ("single1", "single2"), ("loop1", "single1")):
    bad = []
    for k in runs[a]:
        x, y = runs[a][k], runs[b][k]
        if not np.array_equal(x.view(np.uint32), y.view(np.uint32)):
            d = np.abs(x.astype(np.float64) - y)
            bad.append((k, int((d > 0).sum()), float(d.max()), float(np.abs(y).max())))
    print(a, "vs", b, "mismatching tensors:", bad, flush=True)
