"""Pins for oracle/schedule.py (Alg. 2; SURVEY.md §8(c.3) pins 8-9).

Closed form: with F = 1, B = 2, zero latency and
backward-first dispatch, Alg. 2 with pipeline_limit = G_inter reaches the
textbook 1F1B-with-flush bound makespan = (F + B) * (m + P - 1).  The P = 2,
m = 2 trace is checked against a hand simulation."""
import pytest

from oracle import schedule


@pytest.mark.parametrize("P,m", [(2, 2), (2, 4), (4, 8), (4, 32), (4, 64), (8, 16),
                                 (8, 32), (8, 64), (8, 128), (3, 5), (5, 7)])
def test_backward_first_reaches_1f1b_bound(P, m):
    r = schedule.simulate(P, m, policy="backward_first")
    assert r.makespan == 3 * (m + P - 1)


def test_hand_trace_P2_m2():
    """Hand simulation: S0 = F0[0,1] F1[1,2] B0[4,6] B1[7,9]; S1 = F0[1,2] B0[2,4] F1[4,5] B1[5,7]."""
    r = schedule.simulate(2, 2)
    assert r.traces[0] == [("F", 0, 0, 1), ("F", 1, 1, 2), ("B", 0, 4, 6), ("B", 1, 7, 9)]
    assert r.traces[1] == [("F", 0, 1, 2), ("B", 0, 2, 4), ("F", 1, 4, 5), ("B", 1, 5, 7)]
    assert r.makespan == 9


def test_arrival_order_is_slower_at_depth_8():
    """D-19 evidence: arrival-order dispatch loses to backward-first at P = 8
    (regression values from the survey's simulation, Appendix B)."""
    assert schedule.simulate(8, 64, policy="arrival").makespan == 237
    assert schedule.simulate(8, 16, policy="arrival").makespan == 75
    assert schedule.simulate(4, 32, policy="arrival").makespan == 105


def test_stash_profile_P8():
    r = schedule.simulate(8, 64)
    assert r.max_stash == [8, 8, 8, 8, 8, 7, 4, 1]
    assert r.max_inflight == 8


@pytest.mark.parametrize("policy", ["backward_first", "arrival"])
@pytest.mark.parametrize("P,m", [(1, 5), (2, 1), (2, 7), (3, 2), (4, 9), (8, 20)])
@pytest.mark.parametrize("seed", [None, 1, 2, 3])
def test_invariants(policy, P, m, seed):
    """Pin 9: one F and one B per microbatch per stage, backwards ascending,
    F(mu) before B(mu), in-flight <= pipeline_limit, termination."""
    r = schedule.simulate(P, m, policy=policy, seed=seed)
    assert r.max_inflight <= P
    for i in range(P):
        tr = r.traces[i]
        fs = [mb for k, mb, *_ in tr if k == "F"]
        bs = [mb for k, mb, *_ in tr if k == "B"]
        assert sorted(fs) == list(range(m))
        assert bs == list(range(m))          # ascending (D-19)
        assert fs == list(range(m))          # FIFO links => forwards in order
        fend = {mb: e for k, mb, s, e in tr if k == "F"}
        bstart = {mb: s for k, mb, s, e in tr if k == "B"}
        for mb in range(m):
            assert fend[mb] <= bstart[mb]
        # a stage never runs two actions at once
        spans = sorted((s, e) for _, _, s, e in tr)
        for (s0, e0), (s1, e1) in zip(spans, spans[1:]):
            assert e0 <= s1 + 1e-12
    # cross-stage causality: F(i, mu) starts after F(i-1, mu) ends; B(i, mu) after B(i+1, mu)
    for i in range(1, P):
        fprev = {mb: e for k, mb, s, e in r.traces[i - 1] if k == "F"}
        for k, mb, s, e in r.traces[i]:
            if k == "F":
                assert s >= fprev[mb] - 1e-12
    for i in range(P - 1):
        bnext = {mb: e for k, mb, s, e in r.traces[i + 1] if k == "B"}
        for k, mb, s, e in r.traces[i]:
            if k == "B":
                assert s >= bnext[mb] - 1e-12


def test_small_m_injects_min_limit():
    """D-18: m < pipeline_limit injects m microbatches."""
    r = schedule.simulate(4, 2)
    assert r.max_inflight == 2
    assert r.makespan == 3 * (2 + 4 - 1)
