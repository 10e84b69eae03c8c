"""Alg. 2 message-driven inter-layer schedule over virtual workers — oracle
(test infrastructure only).

Follows PAPER.md:383-439 (Alg. 2) literally for one pipeline row of G_inter
stages:

* l.3-9 warm-up: stage 0 pops and forwards ``pipeline_limit`` microbatches,
  sending each output to stage 1 (pipeline_limit = G_inter, PAPER.md:467-470;
  min(limit, m) when m < limit, reading D-18);
* l.11-31 steady state: every stage waits for a message; one from i-1 triggers
  Forward (on the last stage Forward + Backward(1), l.14-16, and the gradient
  goes to i-1); one from i+1 triggers Backward (on stage 0 followed by the
  injection of the next microbatch, l.22-26);
* messages travel over per-link FIFO queues (MPI_Isend/Irecv).

The paper leaves open which landed message is served first when several
have landed (reading D-19): ``policy="backward_first"`` serves gradients
first (FIFO), ``policy="arrival"`` serves the earliest arrival.  G_inter = 1
degenerates to F, loss, B per microbatch with no messages (D-18).

Costs default to F = 1, B = 2 ("the backward pass takes
twice as much time as the forward pass").  Pins (tests/test_oracle_schedule.py):
the 1F1B-flush closed form makespan = (cost_F + cost_B) * (m + P - 1) for the
backward-first policy, the hand-simulated P = 2, m = 2 trace, and the
invariants (one F and one B per microbatch per stage, backwards ascending,
in-flight <= pipeline_limit, termination) under random costs.
"""
from __future__ import annotations

import random
from dataclasses import dataclass, field


@dataclass
class ScheduleResult:
    traces: list                 # per stage: list of (kind, mb, start, end)
    makespan: float
    max_stash: list              # per stage: max microbatches between F and B
    max_inflight: int            # max microbatches injected and not yet backward at stage 0
    order: list = field(default_factory=list)   # global execution order (stage, kind, mb)


def simulate(P: int, m: int, limit: int | None = None, policy: str = "backward_first",
             cost_f: float = 1.0, cost_b: float = 2.0, latency: float = 0.0,
             on_forward=None, on_backward=None, seed: int | None = None) -> ScheduleResult:
    """Run Alg. 2 on P virtual workers for m microbatches.

    ``on_forward(stage, mb)`` / ``on_backward(stage, mb)`` are invoked in a
    causally valid order (every message is produced before it is consumed),
    so payload computations can ride on the simulation.  ``seed`` draws each
    action's cost uniformly in [0.5, 1.5] x nominal (property sweeps)."""
    if P < 1 or m < 0:
        raise ValueError("P >= 1 and m >= 0 required")
    limit = P if limit is None else limit
    if limit < 1:
        raise ValueError("pipeline_limit >= 1 required")
    rng = random.Random(seed) if seed is not None else None

    def cost(kind):
        c = cost_f if kind == "F" else cost_b
        return c * rng.uniform(0.5, 1.5) if rng else c

    traces = [[] for _ in range(P)]
    order = []
    stash = [0] * P
    max_stash = [0] * P
    inflight = 0
    max_inflight = 0

    def run(stage, kind, mb, t):
        nonlocal inflight, max_inflight
        d = cost(kind)
        traces[stage].append((kind, mb, t, t + d))
        order.append((stage, kind, mb))
        if kind == "F":
            if stage == 0:
                inflight += 1
                max_inflight = max(max_inflight, inflight)
            stash[stage] += 1
            max_stash[stage] = max(max_stash[stage], stash[stage])
            if on_forward:
                on_forward(stage, mb)
        else:
            stash[stage] -= 1
            if stage == 0:
                inflight -= 1
            if on_backward:
                on_backward(stage, mb)
        return t + d

    if P == 1:                       # D-18: F, loss, B per microbatch, no messages
        t = 0.0
        for mb in range(m):
            t = run(0, "F", mb, t)
            t = run(0, "B", mb, t)
        return ScheduleResult(traces, t, max_stash, max_inflight, order)

    inbox = [[] for _ in range(P)]   # (arrival, seq, kind, mb); kind 'A' act, 'G' grad
    seq = 0
    free = [0.0] * P
    popped = 0
    expected = [(m if i > 0 else 0) + (m if i < P - 1 else 0) for i in range(P)]
    received = [0] * P

    def send(dst, kind, mb, t):
        nonlocal seq
        inbox[dst].append((t + latency, seq, kind, mb))
        seq += 1

    # Alg. 2 l.3-9: warm-up injection on stage 0
    t = 0.0
    for _ in range(min(limit, m)):
        mb = popped
        popped += 1
        t = run(0, "F", mb, t)
        send(1, "A", mb, t)
    free[0] = t

    # Alg. 2 l.11-31: steady state
    while any(received[i] < expected[i] for i in range(P)):
        best = None
        for i in range(P):
            if not inbox[i]:
                continue
            dec = max(free[i], min(msg[0] for msg in inbox[i]))
            if best is None or dec < best[0]:
                best = (dec, i)
        if best is None:
            raise RuntimeError("Alg. 2 deadlock: messages expected but none in flight")
        tdec, i = best
        landed = [msg for msg in inbox[i] if msg[0] <= tdec]
        if policy == "backward_first" and any(msg[2] == "G" for msg in landed):
            pick = min((msg for msg in landed if msg[2] == "G"), key=lambda x: (x[0], x[1]))
        elif policy in ("backward_first", "arrival"):
            pick = min(landed, key=lambda x: (x[0], x[1]))
        else:
            raise ValueError(f"unknown policy {policy}")
        inbox[i].remove(pick)
        received[i] += 1
        _, _, kind, mb = pick
        t = tdec
        if kind == "A":                                  # l.13-19
            t = run(i, "F", mb, t)
            if i == P - 1:
                t = run(i, "B", mb, t)                   # Backward(1)
                send(i - 1, "G", mb, t)
            else:
                send(i + 1, "A", mb, t)
        else:                                            # l.21-28
            t = run(i, "B", mb, t)
            if i == 0:
                if popped < m:
                    nxt = popped
                    popped += 1
                    t = run(0, "F", nxt, t)
                    send(1, "A", nxt, t)
            else:
                send(i - 1, "G", mb, t)
        free[i] = t
    makespan = max(free)
    return ScheduleResult(traces, makespan, max_stash, max_inflight, order)
