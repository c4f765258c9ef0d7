"""The C++ LBSS selector in libspin.so (csrc/lbss.cpp) against the reference
selector: traces of the reference's own functions (draw_exploration_assignment,
prewarm_destination, plan_exploitation, exploitation_duration -- run_lbss's control
flow, bandit.cpp:248-332, replayed by oracle/ref_shim.cpp ref_lbss_trace) on seeded
goodput tables must be reproduced slot for slot: assignment, prewarm, explore flag.
Golden file: tests/golden/lbss_golden.json (python oracle/make_golden.py lbss)."""
import json
import os

import numpy as np
import pytest

from paper_2503_15921_b200.selector import Lbss

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "lbss_golden.json")


def _cases():
    with open(GOLD) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"n{c['n']}-caps{'-'.join(map(str, c['caps']))}")
def test_cpp_lbss_reproduces_reference_trace(case):
    n, caps, g = case["n"], case["caps"], np.array(case["goodput"])
    sel = Lbss(n, caps, alpha=case["alpha"], beta=case["beta"], seed=case["seed"])
    for t in range(case["slots"]):
        a, explore = sel.next_slot()
        assert a.tolist() == case["assignment"][t], (t, a.tolist(), case["assignment"][t])
        assert sel.prewarm.tolist() == case["prewarm"][t], t
        assert int(explore) == case["explore"][t], t
        for i in range(n):
            if a[i] >= 0:  # the observation model of ref_lbss_trace
                sel.add(i, int(a[i]), g[i, a[i]] * (1.0 + 0.05 * ((i + 3 * int(a[i]) + t) % 5)))
    sel.close()


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
    assert (a0 == 0).sum() <= 3 and (a0 == 1).sum() <= 4
    assert (a0 == -1).sum() == 3  # 10 requests, 7 seats: overflow idles


def test_exploitation_prefers_measured_best_and_cold_arms():
    sel = Lbss(3, [3, 3, 3], alpha=2, beta=1, seed=0)
    sel.add(0, 0, 5.0), sel.add(0, 1, 9.0), sel.add(0, 2, 1.0)
    sel.add(1, 0, 4.0), sel.add(1, 1, 2.0)  # request 1 never tried ssm 2 -> optimistic
    sel.add(2, 2, 7.0), sel.add(2, 0, 3.0), sel.add(2, 1, 3.0)
    assert sel.exploitation().tolist() == [1, 2, 2]


def test_exploitation_matching_under_capacity():
    sel = Lbss(3, [1, 2], alpha=2, beta=1, seed=0)
    for r, (a, b) in enumerate([(10.0, 1.0), (9.0, 8.0), (2.0, 1.0)]):
        sel.add(r, 0, a), sel.add(r, 1, b)
    plan = sel.exploitation()
    assert (plan == 0).sum() == 1
    assert plan.tolist() == [0, 1, 1]  # max total weight: 10 + 8 + 1


def test_rows_roundtrip_and_validation():
    from paper_2503_15921_b200._lib import SpinError

    sel = Lbss(4, [4, 4], alpha=2, beta=1, seed=3)
    sel.add(1, 1, 2.5)
    r = sel.rows()
    assert r[1, 1].tolist() == [2.5, 1.0] and r.sum() == 3.5
    r[2, 0] = [6.0, 2.0]
    sel.set_rows(r)
    assert sel.rows()[2, 0].tolist() == [6.0, 2.0]
    with pytest.raises(SpinError) as ei:
        Lbss(4, [4, 4], alpha=3, beta=2)
    assert ei.value.kind == "ConfigError"
