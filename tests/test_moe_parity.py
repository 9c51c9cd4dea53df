"""Product MoE hooks reproduce the reference's decisions (CPU tier).

tests/golden/moe_fetch.json holds what the reference produced for four
scenarios (make_golden.fetch_plan): residency after place_offloaded/rebalance
(moe.py:155-197, :354-383), including every peer handle (device, base, size,
generation), and the tier + handle of every fetch its decode issued
(moe.py:282-313).  Here the SAME routing trace is fed to
paper_2602_00328_b200.moe.place_offloaded on the B200 runtime (modeled engine,
reference topology constants), and ExpertFetcher.plan must name the same
serving tier and handle for every activated expert of every stage.
"""
import json
import os

import numpy as np
import pytest

from paper_2602_00328_b200 import moe as M
from paper_2602_00328_b200.events import VirtualLoop
from paper_2602_00328_b200.interconnect import LinkKind, LinkSpec, Topology
from paper_2602_00328_b200.memalloc import DeviceSpec, Tier
from paper_2602_00328_b200.runtime import HarvestRuntime

GiB = 1 << 30
G = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "moe_fetch.json")))


def paper_h100_topology(num_peers, peer_capacity):
    """profiles.build_topology(PAPER_H100, ...) (profiles.py:152-181) with the
    paper-h100 constants (profiles.py:58-64)."""
    host_id = num_peers + 1
    devices = [DeviceSpec(0, Tier.LOCAL_HBM, 80 * GiB)]
    links = []
    for pid in range(1, num_peers + 1):
        devices.append(DeviceSpec(pid, Tier.PEER_HBM, peer_capacity))
        links.append(LinkSpec(LinkKind.PEER_LINK, 8.08e-6, 495e9, endpoints=(0, pid)))
        links.append(LinkSpec(LinkKind.HOST_LINK, 15.15e-6, 55e9, endpoints=(pid, host_id)))
    devices.append(DeviceSpec(host_id, Tier.HOST_DRAM, 640 * GiB))
    links.append(LinkSpec(LinkKind.HOST_LINK, 15.15e-6, 55e9, endpoints=(0, host_id)))
    return Topology(devices=devices, links=links), host_id


S_QWEN, S_PHI = 17_301_504, 157_286_400
CASES = {  # name: (model key, fraction, tier, peer capacity, peers)  — make_golden.gen_moe
    "qwen15_b32_peer50": ("qwen1.5-moe-a2.7b", 50, Tier.PEER_HBM, 40 * S_QWEN, 1),
    "qwen15_b32_host100": ("qwen1.5-moe-a2.7b", 100, Tier.HOST_DRAM, 80 * GiB, 1),
    "qwen15_b32_peer100_7donors": ("qwen1.5-moe-a2.7b", 100, Tier.PEER_HBM, 180 * GiB, 7),
    "phi35_b16_peer100_7donors": ("phi-3.5-moe", 100, Tier.PEER_HBM, 11 * GiB, 7),
}


@pytest.mark.parametrize("name", list(CASES))
def test_placement_and_fetch_plan_match_reference(name):
    key, fraction, tier, cap, peers = CASES[name]
    c = G[name]
    L, E, K, S, ct = G["models"][key]
    model = M.MoEProfile(key, L, E, K, S, ct)
    active = [[tuple(x) for x in row] for row in c["active"]]
    trace = M.RoutingTrace(len(active), L, E, active, np.array(c["counts"], dtype=np.int64))
    topo, host_id = paper_h100_topology(peers, cap)
    loop = VirtualLoop()
    rt = HarvestRuntime(loop, topo)
    res = M.ExpertResidency(model)
    M.place_offloaded(loop, rt, model, res, trace, fraction, tier, host_id)
    got = {f"{l},{e}": [ent.tier.value, None if ent.handle is None else list(ent.handle.key())]
           for (l, e), ent in res.entries.items()}
    assert got == c["residency"]
    fetcher = M.ExpertFetcher(rt, model, res, M.ExpertStore(model, host_id, None))
    plan = []
    for layer in range(L):
        for mb in range(len(active)):
            for e, t in fetcher.plan(layer, active[mb][layer]):
                h = fetcher.handles.get((layer, e)) if t == "peer" else None
                plan.append([layer, e, t, None if h is None else list(h.key())])
    assert plan == c["fetches"]
