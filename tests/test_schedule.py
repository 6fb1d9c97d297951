"""NEXT-4 host logic: the training schedule of P:342 / P:204 (paper_2605_13794_b200/train.py)."""
import numpy as np

from paper_2605_13794_b200.train import Schedule, epoch_order, geometric_unlocks


def test_paper_defaults():
    s = Schedule()
    # density control every 500 steps from 2,000 through 20,000
    due = [t for t in range(0, 45001) if s.densify_due(t)]
    assert due[0] == 2000 and due[-1] == 20000 and len(due) == 37
    assert all(b - a == 500 for a, b in zip(due, due[1:]))
    # the LOD gate is disabled inside the window and engaged afterwards
    assert not s.gate_enabled(2000) and not s.gate_enabled(20000) and s.gate_enabled(20001)
    # scoring passes at T1 = 15,000 (stochastic) and T2 = 40,000 (mass); phi after T1
    assert s.scoring_due(15000) == "stochastic" and s.scoring_due(40000) == "mass" and s.scoring_due(15001) is None
    assert not s.phi_active(15000) and s.phi_active(15001)


def test_lmax_geometric_unlock():
    """L_max = 0 until 2,000, +1 at 2,000 * 2^k, capped at K - 1; non-decreasing."""
    s = Schedule(k_levels=6)
    assert geometric_unlocks(s) == [2000, 4000, 8000, 16000, 32000]
    table = {0: 0, 1999: 0, 2000: 1, 3999: 1, 4000: 2, 8000: 3, 15999: 3, 16000: 4, 32000: 5, 10 ** 6: 5}
    for t, lm in table.items():
        assert s.l_max(t) == lm, t
    ts = np.arange(0, 70000, 37)
    vals = [s.l_max(int(t)) for t in ts]
    assert all(b >= a for a, b in zip(vals, vals[1:])) and max(vals) == 5 and min(vals) == 0
    assert Schedule(k_levels=1).l_max(10 ** 6) == 0


def test_scaled_schedule_and_epochs():
    s = Schedule().scaled(0.1)
    assert (s.dc_start, s.dc_end, s.dc_every, s.t1, s.t2, s.unlock_first) == (200, 2000, 50, 1500, 4000, 200)
    o = epoch_order(64, 3, 0)
    assert sorted(o.tolist()) == list(range(64))
    assert not np.array_equal(o, epoch_order(64, 3, 1))
    assert np.array_equal(o, epoch_order(64, 3, 0))
