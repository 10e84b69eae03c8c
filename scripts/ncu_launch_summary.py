"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list of
`bench.py --steps 1 --warmup 1 --e2e-steps 1` (G_inter 1): keep the launches of the timed step
(from the (m+1)-th to just before the (2m+1)-th embed_fwd launch, m = microbatches per step),
write them to OUT.csv and a per-kernel share summary to OUT.json.
m = 0: the log already holds only the timed step (bench.py with AXONN_NVTX=1 under
ncu --nvtx --nvtx-include timed_step/).
Usage: python scripts/ncu_launch_summary.py LOG.csv OUT_PREFIX [m]"""
import csv
import io
import json
import re
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)                      # drop the argument list
    name = re.sub(r"^void ", "", name)
    return name.replace("(anonymous namespace)::", "").replace("axonn::", "")


def main(log, out, m=8):
    text = open(log).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}
    launches = []
    for r in rows[1:]:
        if len(r) < len(hdr) or r[col["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[col["Metric Value"]].replace(",", ""))
        unit = r[col["Metric Unit"]]
        us = v / 1e3 if unit in ("nsecond", "ns") else v * 1e3 if unit in ("msecond", "ms") else v
        launches.append((int(r[col["ID"]]), r[col["Kernel Name"]], us))
    if m == 0:   # the log holds only the timed step (ncu --nvtx-include timed_step/)
        step = launches
    else:
        emb = [i for i, (_, n, _) in enumerate(launches) if "embed_fwd" in n]
        lo, hi = emb[m], emb[2 * m] if len(emb) > 2 * m else len(launches)
        step = launches[lo:hi]
    total = sum(t for _, _, t in step)
    by = {}
    for _, n, t in step:
        k = short(n)
        e = by.setdefault(k, {"ms": 0.0, "launches": 0})
        e["ms"] += t / 1e3
        e["launches"] += 1
    for e in by.values():
        e["share"] = e["ms"] / (total / 1e3)
        e["us_per_launch"] = e["ms"] * 1e3 / e["launches"]
    by = dict(sorted(by.items(), key=lambda kv: -kv[1]["ms"]))
    with open(out + ".csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "us"])
        for i, n, t in step:
            w.writerow([i, short(n), f"{t:.3f}"])
    json.dump({"source": log, "timed_step_launches": len(step), "total_kernel_ms": total / 1e3,
               "note": "ncu serialises launches and runs them cold-cache: compare shares, not times",
               "by_kernel": by}, open(out + ".json", "w"), indent=1)
    print(json.dumps({k: round(v["share"], 4) for k, v in by.items()}, indent=0))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 8)
