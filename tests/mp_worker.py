"""Worker for the multi-GPU parity tests (launched by torchrun, one rank per GPU).

Writes the seeded parity weights of its stage, runs batches through the C-ABI
and dumps losses / gradients / updated weights to <out>/rank<r>.npz."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")   # before any CUDA context


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--g-inter", type=int, required=True)
    ap.add_argument("--g-data", type=int, required=True)
    ap.add_argument("--mb", type=int, default=2)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--cfg", default="tiny")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--offload", type=int, default=0)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--loss-scale", type=float, default=1.0)
    ap.add_argument("--inf-rank", type=int, default=-1,
                    help="after step 0's run_batch this rank writes one inf gradient (D-12 skip)")
    ap.add_argument("--balance", action="store_true", help="stage_balance (reading D-21b)")
    ap.add_argument("--speed", default=None,
                    help="with --balance: 'calibrate' or comma-separated stage speeds (reading D-21c)")
    ap.add_argument("--half-accum", action="store_true",
                    help="grad_accum_fp32 = 0: weight matrices accumulate in the half gradient (D-38)")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import torch
    from paper_2110_13005_b200 import dist as D
    from paper_2110_13005_b200.engine import T_GRAD, T_GRAD32, T_MASTER, AxoNN, AxoNNError
    from synth import init_params, markov_tokens
    cfgs = {"tiny": dict(n_layers=2, hidden=64, heads=2, seq_len=32, vocab=256),
            "tiny4": dict(n_layers=4, hidden=64, heads=2, seq_len=32, vocab=256),
            "mini": dict(n_layers=4, hidden=256, heads=4, seq_len=128, vocab=1024),
            "tinyv": dict(n_layers=2, hidden=64, heads=2, seq_len=32, vocab=1024),
            "tiny4v": dict(n_layers=4, hidden=64, heads=2, seq_len=32, vocab=2048)}
    cfg = cfgs[a.cfg]
    rank, world, local = D.env_rank_world()
    if "AXONN_WATCHDOG_S" in os.environ:   # stagger so every rank reports its own state
        os.environ["AXONN_WATCHDOG_S"] = str(float(os.environ["AXONN_WATCHDOG_S"]) + 15 * rank)
    torch.cuda.set_device(local)
    D.init_process_group(rank, world)
    nid = D.share_unique_id(rank, world, D.nccl_unique_id)
    eng = AxoNN(a.g_inter, a.g_data, a.mb, **cfg, rank=rank, world_size=world, device=local,
                nccl_id=nid, offload=bool(a.offload), bucket_elems=5000, coarsen_k=2,
                dtype=a.dtype, loss_scale=a.loss_scale, grad_accum_fp32=not a.half_accum,
                stage_balance="calibrate" if (a.balance and a.speed == "calibrate") else a.balance,
                stage_speed=[float(x) for x in a.speed.split(",")]
                if (a.speed and a.speed != "calibrate") else None)
    params = init_params(cfg["n_layers"], cfg["hidden"], cfg["seq_len"], cfg["vocab"], seed=42)
    names = [n for n, _, _ in eng.tensors()]
    eng.write_all(T_MASTER, {n: params[n] for n in names})
    out = {"bounds": np.array(eng.partition() if a.balance else [])}
    if eng.stage_speed is not None:
        out["speed"] = np.array(eng.stage_speed)
    for step in range(a.steps):
        tok = markov_tokens(a.batch, cfg["seq_len"], cfg["vocab"], seed=7 + step)
        loss = eng.run_batch(tok)
        out[f"loss{step}"] = np.array(loss)
        if step == 0:
            for idx, n in enumerate(names):
                try:   # with --half-accum the weight matrices have no fp32 accumulator
                    out["g32." + n] = eng.read(T_GRAD32, idx)
                except AxoNNError:
                    assert a.half_accum, n
            for n, v in eng.read_all(T_GRAD).items():
                out["g16." + n] = v
        if step == 0 and a.inf_rank >= 0:
            before = eng.read_all(T_MASTER)
            if rank == a.inf_rank:
                g = eng.read(T_GRAD, 0)
                g.reshape(-1)[g.size // 2] = np.inf
                eng.write(T_GRAD, 0, g)
            try:
                eng.optimizer_step()
                out["skipped"] = np.array(0)
            except AxoNNError as e:
                out["skipped"] = np.array(1 if e.status == "NONFINITE" else -1)
            after = eng.read_all(T_MASTER)
            out["unchanged"] = np.array(all(np.array_equal(before[n], after[n]) for n in before))
            eng.run_batch(tok)   # the skipped step is redone on the same batch
        eng.optimizer_step()
    for n, v in eng.read_all(T_MASTER).items():
        out["theta." + n] = v
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), **out)
    D.barrier(world)
    eng.close()


if __name__ == "__main__":
    main()
