"""Property tests of the runtime (SPEC.md:181-186 invariants) on random op
sequences over the modeled engine: exact accounting after every op,
drain-before-free / invalidate-before-notify on the log (verify.py:25-69),
no runtime-initiated transfers, and stale handles never succeed."""
import hypothesis.strategies as st
from hypothesis import HealthCheck, given, settings

from paper_2602_00328_b200 import runtime as R
from paper_2602_00328_b200.events import VirtualLoop
from paper_2602_00328_b200.memalloc import Segment, check_invariants
from tests import refcheck
from tests.test_runtime_parity import topo

MiB = 1 << 20

op = st.one_of(
    st.tuples(st.just("alloc"), st.integers(1, 24 * MiB), st.sampled_from([None, [1], [2]])),
    st.tuples(st.just("free"), st.integers(0, 50)),
    st.tuples(st.just("revoke"), st.integers(0, 50)),
    st.tuples(st.just("read"), st.integers(0, 50)),
    st.tuples(st.just("reclaim"), st.sampled_from([1, 2]), st.integers(0, 64 * MiB)),
    st.tuples(st.just("avail"), st.sampled_from([1, 2]), st.integers(0, 64 * MiB)),
    st.tuples(st.just("time"), st.floats(0, 1e-3)),
)


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.lists(op, min_size=1, max_size=60), st.sampled_from(list(R.PolicyKind)))
def test_random_schedules_keep_invariants(ops, kind):
    loop = VirtualLoop()
    pol = R.Policy(kind, fairness_budget_bytes_per_s=64 * MiB / 1e-3, fairness_burst_bytes=32 * MiB,
                   stability_window_s=1e-3, stability_max_revocations=2)
    rt = R.HarvestRuntime(loop, topo([(64 * MiB, 0, 0), (48 * MiB, 4 * MiB, 2 * MiB)]), policy=pol)
    handles, called = [], []
    for o in ops:
        k = o[0]
        if k == "alloc":
            h = rt.harvest_alloc(o[1], R.AllocationHints(preferred_devices=o[2]))
            if h is not None:
                handles.append(h)
                rt.harvest_register_cb(h, lambda hh, r: called.append(hh))
        elif k in ("free", "revoke", "read") and handles:
            h = handles[o[1] % len(handles)]
            if k == "free":
                live = rt.lookup(h) is not None and rt.placement[h.key()].state == R._State.LIVE
                try:
                    rt.harvest_free(h)
                    assert live
                except R.StaleHandleError:
                    assert not live
            elif k == "revoke":
                rt.revoke(h, R.RevokeReason.POLICY)
            elif rt.is_live(h):
                rt.write_peer(h, "t", 1)
                rt.app_transfer(src=(h.device_id, Segment(h.base, h.size)), dst=(0, Segment(0, h.size)),
                                size=h.size, tag="t", handle=h)
        elif k == "reclaim":
            rt.external_reclaim(o[1], o[2])
        elif k == "avail":
            rt.set_availability(o[1], o[2])
        elif k == "time":
            loop.run(until=loop.now + o[1])
        # exact accounting after every op
        for dev, stt in rt.devices.items():
            check_invariants(stt)
            held = sum(e.handle.size for e in rt.placement.values() if e.handle.device_id == dev)
            assert rt.occupied_bytes(dev) == held
    loop.run()
    assert not rt.placement or all(e.state == R._State.LIVE for e in rt.placement.values())
    assert refcheck.verify_release_ordering(loop.log) == []
    assert refcheck.verify_no_runtime_writeback(loop.log) == []
    for h in called:  # a revoked handle is dead for every later operation
        assert not rt.is_live(h)
        try:
            rt.harvest_free(h)
            raise AssertionError("stale handle accepted")
        except R.StaleHandleError:
            pass


def test_fairness_tokens_not_spent_when_donor_commit_fails():
    """a donor HBM shortfall (pool.commit fails after the
    best-fit decision) returns None like NoCapacity and must not drain the
    client's fairness budget; the next allocation still fits the burst."""
    from paper_2602_00328_b200 import _native as N
    GiB = 1 << 30

    class FlakyPool:
        def __init__(self):
            self.fail = True

        def commit(self, base, size):
            if self.fail:
                raise N.HarvestNativeError(-1000 - 2, "hv_pool_commit")

        def decommit(self, base, size):
            pass

    loop = VirtualLoop()
    pool = FlakyPool()
    pol = R.Policy(R.PolicyKind.FAIRNESS, fairness_budget_bytes_per_s=0.0, fairness_burst_bytes=float(GiB))
    rt = R.HarvestRuntime(loop, topo([(4 * GiB, 0, 0)]), pol, pools={1: pool})
    hints = R.AllocationHints(client_id="c")
    assert rt.harvest_alloc(GiB, hints) is None          # commit failed
    pool.fail = False
    h = rt.harvest_alloc(GiB, hints)                      # the whole burst is still there
    assert h is not None
    assert rt.harvest_alloc(1, hints) is None             # and now it is spent
