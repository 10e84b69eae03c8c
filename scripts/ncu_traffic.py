"""Summarise an `ncu --set full` capture of the K1 linear-layer GEMM launches into
profiles/<round>/k1_traffic.json: per launch duration, DRAM bytes (dram__bytes_read.sum +
dram__bytes_write.sum), the algorithmic bytes of the launch (A + B read, C written, plus the
fused epilogue's extra operand), and the tensor-pipe utilisation.  bench.py reports the
average as roofline.traffic.  Usage: python scripts/ncu_traffic.py REPORT.ncu-rep OUT.json [M tokens per microbatch]"""
import csv
import io
import json
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def main(rep, out, M=4096):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, name):
        i = col[name]
        v = float(r[i].replace(",", ""))
        return v * UNITS.get(units[i], 1)

    launches = []
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        if "gemm_bf16_tcgen05_pair" not in name:
            continue
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        rec = {"kernel": name.split("(")[0], "grid": r[col["launch__grid_size"]],
               "us": val(r, "gpu__time_duration.sum") * 1e6, "dram_read": rd, "dram_write": wr,
               "dram_total": rd + wr}
        for k in ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                  "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                  "lts__throughput.avg.pct_of_peak_sustained_elapsed"):
            if k in col and rows[2][col[k]] not in ("", "n/a"):
                try:
                    rec[k] = float(r[col[k]].replace(",", ""))
                except ValueError:
                    pass
        launches.append(rec)
    # algorithmic bytes of the 15 K1 launches of one 1-layer microbatch (issue order of
    # model_exec.cpp: forward qkv, proj, fc1, fc2, head; backward head wgrad, head dgrad, then
    # fc2 wgrad, fc2 dgrad, fc1 wgrad, fc1 dgrad, proj wgrad, proj dgrad, qkv wgrad, qkv dgrad)
    # at M tokens, width h, vocab V; bf16 2 B, fp32 gradient 4 B (first microbatch: store only)
    h, V = 2048, 51200
    b2, f4 = 2, 4
    alg = [("fwd qkv", b2 * (M * h + 3 * h * h + M * 3 * h)),
           ("fwd proj +resid", b2 * (M * h + h * h + 2 * M * h)),
           ("fwd fc1 +gelu +pre", b2 * (M * h + 4 * h * h + 2 * M * 4 * h)),
           ("fwd fc2 +resid", b2 * (M * 4 * h + 4 * h * h + 2 * M * h)),
           ("fwd head", b2 * (M * h + V * h + M * V)),
           ("wgrad head", b2 * (M * V + M * h) + f4 * V * h),
           ("dgrad head", b2 * (M * V + V * h + M * h)),
           ("wgrad fc2", b2 * (M * h + M * 4 * h) + f4 * h * 4 * h),
           ("dgrad fc2 *gelu'", b2 * (M * h + 4 * h * h + 2 * M * 4 * h)),
           ("wgrad fc1", b2 * (M * 4 * h + M * h) + f4 * 4 * h * h),
           ("dgrad fc1", b2 * (M * 4 * h + 4 * h * h + M * h)),
           ("wgrad proj", b2 * (2 * M * h) + f4 * h * h),
           ("dgrad proj", b2 * (M * h + h * h + M * h)),
           ("wgrad qkv", b2 * (M * 3 * h + M * h) + f4 * 3 * h * h),
           ("dgrad qkv", b2 * (M * 3 * h + 3 * h * h + M * h))]
    if len(launches) == len(alg):
        for l, (name, a) in zip(launches, alg):
            l["gemm"] = name
            l["algorithmic_bytes"] = a
            l["dram_over_algorithmic"] = l["dram_total"] / a
    avg = sum(l["dram_total"] for l in launches) / max(len(launches), 1)
    res = {"report": rep, "hidden": h, "tokens": M, "launches": launches, "n": len(launches),
           "dram_bytes_per_launch_avg": avg}
    if len(launches) == len(alg):
        res["algorithmic_bytes_per_launch_avg"] = sum(a for _, a in alg) / len(alg)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "launches"}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 4096)
