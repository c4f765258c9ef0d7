"""Host LBSS selector (selector.py) against the reference bandit's semantics."""
import numpy as np

from paper_2503_15921_b200.selector import Lbss


def test_epoch_schedule_matches_reference():
    # phase_of_slot (bandit.cpp:33-52): alpha explore slots, then 2^k exploit slots, k = 1, 2, ...
    sel = Lbss(6, [6, 6], alpha=4, beta=2, seed=1)
    flags = [sel.next_slot()[1] for _ in range(4 + 2 + 4 + 4 + 4 + 8)]
    assert flags == [True] * 4 + [False] * 2 + [True] * 4 + [False] * 4 + [True] * 4 + [False] * 8


def test_exploration_chunks_hold_assignment_and_respect_capacity():
    sel = Lbss(10, [3, 4], alpha=4, beta=2, seed=7)
    a0, _ = sel.next_slot()
    a1, _ = sel.next_slot()
    assert np.array_equal(a0, a1)  # a chunk keeps its draw for beta slots
    for a in (a0,):
        assert (a == 0).sum() <= 3 and (a == 1).sum() <= 4
        assert (a == -1).sum() == 3  # 10 requests, 7 seats: overflow idles


def test_exploitation_prefers_measured_best_and_cold_arms():
    sel = Lbss(3, [3, 3, 3], alpha=2, beta=1, seed=0)
    sel.add(0, 0, 5.0), sel.add(0, 1, 9.0), sel.add(0, 2, 1.0)
    sel.add(1, 0, 4.0), sel.add(1, 1, 2.0)  # request 1 never tried ssm 2 -> optimistic
    sel.add(2, 2, 7.0), sel.add(2, 0, 3.0), sel.add(2, 1, 3.0)
    plan = sel.exploitation()
    assert plan.tolist() == [1, 2, 2]


def test_exploitation_matching_under_capacity():
    sel = Lbss(3, [1, 2], alpha=2, beta=1, seed=0)
    for r, (a, b) in enumerate([(10.0, 1.0), (9.0, 8.0), (2.0, 1.0)]):
        sel.add(r, 0, a), sel.add(r, 1, b)
    plan = sel.exploitation()
    assert (plan == 0).sum() == 1
    assert plan.tolist() == [0, 1, 1]  # max total weight: 10 + 8 + 1
