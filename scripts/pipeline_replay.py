"""Replay of a measured pipeline (the discrete-event view of Alg. 2).

Reads the per-op timelines the library writes with AXONN_TIMELINE (one CSV per rank: every
Forward / Backward of the batch with its start and end on the stage's compute stream, and the
time each message was observed landed), takes each stage's measured F and B durations per
microbatch, and re-runs Alg. 2 (backward-first among landed messages, D-19;
stage 0 injects min(limit, m) microbatches, then one after each backward; the last stage runs
F and B back to back) as a discrete-event simulation with zero-latency messages.  The
simulated makespan is what the measured op durations allow; the measured span minus it is the
time lost to message hand-off and dispatch.  A second replay gives every stage the same
(median) op times: the gap between the two is the stage imbalance.

Analysis tooling only (not imported by the library, the tests or bench.py).

    python scripts/pipeline_replay.py profiles/r2/d21d_rejected/timeline_16l_4x1/gi4
"""
import csv
import glob
import heapq
import json
import statistics
import sys


def load(prefix):
    stages = {}
    for path in sorted(glob.glob(prefix + ".rank*.csv")):
        ops = {"F": {}, "B": {}}
        t0, t1 = None, None
        for r in csv.DictReader(open(path)):
            if r["kind"] in ("F", "B"):
                a, b = float(r["start_ms"]), float(r["end_ms"])
                ops[r["kind"]][int(r["mb"])] = b - a
                t0 = a if t0 is None else min(t0, a)
                t1 = b if t1 is None else max(t1, b)
                st = int(r["stage"])
        stages[st] = {"F": ops["F"], "B": ops["B"], "span": (t0, t1)}
    return [stages[i] for i in sorted(stages)]


def replay(costF, costB, m, limit=None):
    """Alg. 2 event simulation; costF[i][mb], costB[i][mb] in ms; returns the makespan and the
    per-stage busy time."""
    P = len(costF)
    limit = P if limit is None else limit
    busy = [0.0] * P
    idle = [True] * P
    landed = [[] for _ in range(P)]      # (kind, land time, mb)
    ev = []                              # (time, seq, what, stage, kind, mb)
    seq = [0]
    end_all = [0.0]

    def push(t, what, stage, kind=None, mb=None):
        seq[0] += 1
        heapq.heappush(ev, (t, seq[0], what, stage, kind, mb))

    injected = min(limit, m)
    for mb in range(injected):
        push(0.0, "land", 0, "F", mb)

    def start(i, t):
        nonlocal injected
        if not idle[i] or not landed[i]:
            return
        grads = [x for x in landed[i] if x[0] == "B"]
        pick = min(grads or landed[i], key=lambda x: (x[1], x[2]))   # backward first, FIFO
        landed[i].remove(pick)
        kind, _, mb = pick
        idle[i] = False
        if kind == "F":
            end = t + costF[i][mb]
            busy[i] += costF[i][mb]
            if i == P - 1:   # l.14-16: the last stage runs Backward at once
                end += costB[i][mb]
                busy[i] += costB[i][mb]
                if i > 0:
                    push(end, "land", i - 1, "B", mb)
                elif injected < m:
                    push(end, "land", 0, "F", injected)
                    injected += 1
            else:
                push(end, "land", i + 1, "F", mb)
        else:
            end = t + costB[i][mb]
            busy[i] += costB[i][mb]
            if i > 0:
                push(end, "land", i - 1, "B", mb)
            elif injected < m:   # l.22-26: stage 0 injects the next microbatch
                push(end, "land", 0, "F", injected)
                injected += 1
        push(end, "free", i)
        end_all[0] = max(end_all[0], end)

    while ev:
        t = ev[0][0]
        while ev and ev[0][0] == t:      # every event at time t before any choice
            _, _, what, i, kind, mb = heapq.heappop(ev)
            if what == "land":
                landed[i].append((kind, t, mb))
            else:
                idle[i] = True
        for i in range(P):
            start(i, t)
    return end_all[0], busy


def main(prefix):
    st = load(prefix)
    P = len(st)
    m = len(st[0]["F"])
    costF = [[s["F"][mb] for mb in range(m)] for s in st]
    costB = [[s["B"][mb] for mb in range(m)] for s in st]
    measured = max(s["span"][1] for s in st) - min(s["span"][0] for s in st)
    sim, busy = replay(costF, costB, m)
    medF = statistics.median(x for row in costF for x in row)
    medB = statistics.median(x for row in costB for x in row)
    flat, _ = replay([[medF] * m] * P, [[medB] * m] * P, m)
    out = {
        "timeline": prefix, "G_inter": P, "m": m,
        "stage_F_median_ms": [round(statistics.median(r), 3) for r in costF],
        "stage_B_median_ms": [round(statistics.median(r), 3) for r in costB],
        "measured_span_ms": round(measured, 1),
        "replay_measured_ops_ms": round(sim, 1),
        "replay_uniform_ops_ms": round(flat, 1),
        "closed_form_uniform_ms": round((medF + medB) * (m + P - 1), 1),
        "lost_to_messages_and_dispatch": round(1 - sim / measured, 4),
        "lost_to_stage_imbalance": round(1 - flat / sim, 4) if sim > 0 else None,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1])
