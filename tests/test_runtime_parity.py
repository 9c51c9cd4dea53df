"""The B200 runtime reproduces the reference's decisions exactly.

tests/golden/runtime_scenarios.json was produced by running the reference
HarvestRuntime (runtime.py:119-487) on scripted op sequences (allocations
under the four policies, frees, revocations, reads that must drain,
LRU/FIFO reclaim, availability timelines).  Here the same scripts are replayed
on paper_2602_00328_b200.runtime.HarvestRuntime over its VirtualLoop + modeled
engine and every return value, callback and log record must match; the
reference's own checkers (restated in tests/refcheck.py) must find no
ordering violations.
"""
import json
import os

import pytest

from paper_2602_00328_b200 import runtime as R
from paper_2602_00328_b200.events import VirtualLoop
from paper_2602_00328_b200.interconnect import LinkKind, LinkSpec, Topology
from paper_2602_00328_b200.memalloc import DeviceSpec, Segment, Tier
from tests import refcheck

GiB = 1 << 30
HERE = os.path.dirname(os.path.abspath(__file__))
SCEN = json.load(open(os.path.join(HERE, "golden", "runtime_scenarios.json")))["scenarios"]


def topo(peers, hops=None, host_cap=64 * GiB):
    devices = [DeviceSpec(0, Tier.LOCAL_HBM, 16 * GiB)]
    links = []
    hid = len(peers) + 1
    for i, (cap, reserved, headroom) in enumerate(peers, start=1):
        devices.append(DeviceSpec(i, Tier.PEER_HBM, cap, reserved=reserved, headroom=headroom))
        links.append(LinkSpec(LinkKind.PEER_LINK, 1e-6, 100e9, endpoints=(0, i),
                              hops=(hops or {}).get(str(i), (hops or {}).get(i, 1))))
        links.append(LinkSpec(LinkKind.HOST_LINK, 10e-6, 10e9, endpoints=(i, hid)))
    devices.append(DeviceSpec(hid, Tier.HOST_DRAM, host_cap))
    links.append(LinkSpec(LinkKind.HOST_LINK, 10e-6, 10e9, endpoints=(0, hid)))
    return Topology(devices=devices, links=links)


def policy_of(s):
    budget, burst, window, maxrev = s["policy_params"]
    return R.Policy(R.PolicyKind(s["policy"]),
                    fairness_budget_bytes_per_s=float("inf") if budget is None else budget,
                    fairness_burst_bytes=burst, stability_window_s=window, stability_max_revocations=maxrev)


def hkey(h):
    return None if h is None else [h.device_id, h.base, h.size, h.generation]


LOG_KINDS = ("alloc", "alloc_nocapacity", "free_begin", "revoke_begin", "invalidate", "callback", "free",
             "reclaim", "availability_step", "transfer_start", "transfer_complete")
KEEP = ("device", "base", "size", "gen", "reason", "cause", "client", "amount", "revoked", "freed", "level",
        "src", "dst", "handle", "initiator")


def log_of(loop):
    out = []
    for r in loop.log:
        if r.kind not in LOG_KINDS:
            continue
        d = {k: (list(v) if isinstance(v, tuple) else v) for k, v in r.data.items() if k in KEEP}
        out.append([r.kind, d])
    return out


def replay(s):
    loop = VirtualLoop()
    rt = R.HarvestRuntime(loop, topo(s["peers"], s["hops"]), policy=policy_of(s))
    handles, results, cbs = {}, [], []
    for op in s["script"]:
        kind = op[0]
        if kind == "time":
            loop.run(until=op[1])
            results.append(None)
        elif kind == "alloc":
            _, name, size, pref, client = op
            h = rt.harvest_alloc(size, R.AllocationHints(preferred_devices=pref, client_id=client))
            handles[name] = h
            if h is not None:
                rt.harvest_register_cb(h, lambda hh, reason, name=name: cbs.append([name, reason.value]))
            results.append(hkey(h))
        elif kind in ("free", "revoke", "touch", "read", "lookup") and handles.get(op[1]) is None:
            results.append("none")
        elif kind == "free":
            try:
                rt.harvest_free(handles[op[1]])
                results.append("ok")
            except R.StaleHandleError:
                results.append("stale")
        elif kind == "revoke":
            rt.revoke(handles[op[1]], R.RevokeReason(op[2]))
            results.append("ok")
        elif kind == "touch":
            rt.touch(handles[op[1]])
            results.append("ok")
        elif kind == "reclaim":
            results.append([hkey(h) for h in rt.external_reclaim(op[1], op[2], order=op[3])])
        elif kind == "availability":
            rt.apply_availability(op[1], [tuple(x) for x in op[2]])
            results.append("ok")
        elif kind == "read":
            h = handles[op[1]]
            if rt.is_live(h):
                rt.write_peer(h, ("t", op[1]), 1)
                rt.app_transfer(src=(h.device_id, Segment(h.base, h.size)), dst=(0, Segment(0, h.size)),
                                size=h.size, tag=("t", op[1]), handle=h)
                results.append("issued")
            else:
                results.append("miss")
        elif kind == "run":
            loop.run()
            results.append(None)
        elif kind == "lookup":
            results.append(rt.is_live(handles[op[1]]))
        elif kind == "state":
            results.append({str(d): [rt.occupied_bytes(d), rt.harvestable(d)]
                            for d in rt.devices if rt.devices[d].spec.tier == Tier.PEER_HBM})
    loop.run()
    return rt, loop, results, cbs


def _norm(x):
    return json.loads(json.dumps(x))


@pytest.mark.parametrize("s", SCEN, ids=[s["name"] for s in SCEN])
def test_scenario_matches_reference(s):
    rt, loop, results, cbs = replay(s)
    assert _norm(results) == s["results"]
    assert _norm(cbs) == s["callbacks"]
    assert _norm(log_of(loop)) == s["log"]
    assert refcheck.verify_release_ordering(loop.log) == s["release_violations"] == []
    assert refcheck.verify_no_runtime_writeback(loop.log) == []
    for st in rt.devices.values():
        from paper_2602_00328_b200.memalloc import check_invariants
        check_invariants(st)


def test_spec_examples_runtime():
    """SPEC.md:132-170 examples, restated."""
    loop = VirtualLoop()
    rt = R.HarvestRuntime(loop, topo([(10 * GiB, 0, 0), (2 * GiB, 0, 0)]))
    h = rt.harvest_alloc(3 * GiB // 2)
    assert h.device_id == 2                                  # smaller leftover across devices
    assert rt.harvest_alloc(11 * GiB) is None                # larger than every peer
    h1 = rt.harvest_alloc(1 << 20, R.AllocationHints(preferred_devices=[1]))
    assert h1.device_id == 1                                 # hint honoured
    rt.harvest_free(h1)
    loop.run()
    with pytest.raises(R.StaleHandleError):
        rt.harvest_free(h1)                                  # free twice -> stale
    fired = []
    rt.harvest_register_cb(h, lambda hh, r: fired.append(("first", r)))
    rt.harvest_register_cb(h, lambda hh, r: fired.append(("second", r)))
    rt.revoke(h, R.RevokeReason.POLICY)
    rt.revoke(h, R.RevokeReason.POLICY)                      # idempotent
    loop.run()
    assert fired == [("second", R.RevokeReason.POLICY)]
    assert rt.harvestable(1) == 10 * GiB and rt.harvestable(2) == 2 * GiB
    with pytest.raises(ValueError):
        rt.harvest_alloc(0)
    with pytest.raises(ValueError):
        rt.external_reclaim(1, 1, order="mru")
    assert rt.external_reclaim(1, 0) == []


def test_fairness_zero_budget_and_locality():
    loop = VirtualLoop()
    rt = R.HarvestRuntime(loop, topo([(1 * GiB, 0, 0)]),
                          policy=R.Policy(R.PolicyKind.FAIRNESS, fairness_budget_bytes_per_s=0.0))
    assert rt.harvest_alloc(1) is None
    rt2 = R.HarvestRuntime(VirtualLoop(), topo([(1 * GiB, 0, 0), (4 * GiB, 0, 0)], hops={1: 2, 2: 1}),
                           policy=R.Policy(R.PolicyKind.LOCALITY))
    assert rt2.harvest_alloc(1 << 20).device_id == 2
