"""Availability processes (traces.py:155-213) restated in churn.py produce the
reference's exact timelines (tests/golden/traces.json), and a modeled churn
replay on the runtime keeps the reference's release ordering."""
import json
import os

from paper_2602_00328_b200.churn import AvailabilityProcess, availability_from_trace, markov_availability

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "traces.json")
GB = 1 << 30


def test_markov_matches_reference():
    g = json.load(open(G))
    a = markov_availability([0, 45 * GB, 90 * GB, 180 * GB], [0.05] * 4, seed=5, horizon=2.0)
    assert [list(x) for x in a.steps] == [list(x) for x in g["markov_c5"]]
    b = markov_availability([10, 20], [10.0, 10.0], seed=1, horizon=100.0)
    assert [list(x) for x in b.steps] == [list(x) for x in g["markov_two_level"]]


def test_spec_examples():
    # SPEC.md:126-128 (availability_from_trace) and :135-137 (markov)
    a = availability_from_trace([(0.0, 0.3), (10.0, 0.3)], 80 * GB)
    assert all(v == int(80 * GB * 0.7) for _, v in a.steps)
    b = availability_from_trace([(0.0, 1.0)], 80 * GB)
    assert b.steps[0][1] == 0
    c = markov_availability([7], [1.0], seed=3, horizon=10.0)
    assert {v for _, v in c.steps} == {7}
    p = AvailabilityProcess(steps=[(0.0, 5), (2.0, 1)])
    assert p.level_at(1.0) == 5 and p.level_at(2.0) == 1


def test_modeled_churn_release_ordering():
    from paper_2602_00328_b200 import runtime as R
    from paper_2602_00328_b200.events import VirtualLoop
    from tests import refcheck
    from tests.test_runtime_parity import topo
    loop = VirtualLoop()
    rt = R.HarvestRuntime(loop, topo([(64 << 20, 0, 0), (64 << 20, 0, 0)]))
    hs = [rt.harvest_alloc(4 << 20) for _ in range(20)]
    assert all(h is not None for h in hs)
    proc = markov_availability([0, 16 << 20, 64 << 20], [0.01] * 3, seed=5, horizon=0.2)
    for dev in (1, 2):
        rt.apply_availability(dev, proc.steps)
    loop.run()
    assert loop.log.of_kind("revoke_begin")
    assert refcheck.verify_release_ordering(loop.log) == []
