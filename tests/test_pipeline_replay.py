"""scripts/pipeline_replay.py (the DESIGN §8 replay of Alg. 2 on measured op times) pinned
against the oracle's Alg. 2 simulator and the 1F1B closed form (test infrastructure)."""
import os
import sys

import pytest

from oracle import schedule

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
from pipeline_replay import replay  # noqa: E402


@pytest.mark.parametrize("P,m", [(1, 1), (1, 5), (2, 2), (2, 7), (4, 4), (4, 9), (3, 64)])
def test_uniform_costs_match_oracle_and_closed_form(P, m):
    f, b = 1.0, 2.0
    mk, busy = replay([[f] * m] * P, [[b] * m] * P, m)
    assert mk == pytest.approx((f + b) * (m + P - 1))
    assert mk == pytest.approx(schedule.simulate(P, m, cost_f=f, cost_b=b).makespan)
    assert all(x == pytest.approx(m * (f + b)) for x in busy)


def test_stage_dependent_costs_by_hand():
    """P = 2, m = 2, stage 0: F 1, B 2; stage 1: F 2, B 3 (hand-simulated Alg. 2):
    s0 F0 [0,1], F1 [1,2]; s1 F0+B0 [1,6]; s0 B0 [6,8]; s1 F1+B1 [6,11]; s0 B1 [11,13]."""
    mk, busy = replay([[1.0, 1.0], [2.0, 2.0]], [[2.0, 2.0], [3.0, 3.0]], 2)
    assert mk == pytest.approx(13.0)
    assert busy == pytest.approx([6.0, 10.0])


def test_slowest_stage_sets_the_steady_state():
    """m >> P: the makespan approaches m * (F + B) of the slowest stage."""
    P, m = 4, 200
    costF = [[1.0] * m for _ in range(P)]
    costB = [[2.0] * m for _ in range(P)]
    costF[2] = [1.2] * m
    costB[2] = [2.4] * m
    mk, _ = replay(costF, costB, m)
    assert m * 3.6 <= mk <= m * 3.6 + (P - 1) * 3.6 + 1e-9
