"""Differential test against the reference runtime itself, on fresh random
scripts (not the committed goldens): every return value, callback and
event-log record of paper_2602_00328_b200.runtime must equal harvestsim's
(runtime.py:119-487) for 100 new op sequences over the four placement
policies.  CPU only; runs when the unmodified reference is installed under
baseline/_ref (pip install of /root/reference/pkg) and is
skipped otherwise.  The GPU box never needs it.
"""
import os
import random
import sys
import zlib

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(os.path.dirname(HERE), "baseline", "_ref")
pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "harvestsim")),
                                reason="reference not installed under baseline/_ref")


def _golden_tools():
    os.environ["HARVEST_REFERENCE"] = REF
    sys.path.insert(0, os.path.join(HERE, "golden"))
    import make_golden   # runs the reference (harvestsim) from baseline/_ref
    return make_golden


CONFIGS = [
    ("bestfit", "BestFit", [None, None, 10.0, 3], [(64 << 20, 0, 0), (40 << 20, 0, 0), (100 << 20, 8 << 20, 4 << 20)],
     None),
    ("locality", "Locality", [None, None, 10.0, 3], [(64 << 20, 0, 0)] * 3, {1: 2, 2: 1, 3: 3}),
    ("fairness", "Fairness", [8 << 20, 24 << 20, 10.0, 3], [(128 << 20, 0, 0)] * 2, None),
    ("stability", "Stability", [None, None, 2.0, 2], [(64 << 20, 0, 0)] * 3, None),
]


@pytest.mark.parametrize("seed", range(25))
@pytest.mark.parametrize("cfg", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_random_script_matches_reference(cfg, seed):
    mg = _golden_tools()
    from tests import test_runtime_parity as P
    name, kind, params, peers, hops = cfg
    ref_runtime = mg.runtime
    K = ref_runtime.PolicyKind
    budget, burst, window, maxrev = params
    ref_policy = ref_runtime.Policy(K(kind), fairness_budget_bytes_per_s=float("inf") if budget is None else budget,
                                    fairness_burst_bytes=burst,
                                    stability_window_s=window, stability_max_revocations=maxrev)
    script = mg.random_script(random.Random(zlib.crc32(f"diff-{name}-{seed}".encode())), 150, peers)
    want = mg.run_script(ref_policy, peers, script, hops)
    s = {"peers": peers, "hops": hops, "policy": kind, "policy_params": params, "script": script}
    rt, loop, results, cbs = P.replay(s)
    assert P._norm(results) == P._norm(want["results"])
    assert P._norm(cbs) == P._norm(want["callbacks"])
    assert P._norm(P.log_of(loop)) == P._norm(want["log"])
    assert want["release_violations"] == [] and want["writeback_violations"] == []


MOE_CASES = [  # (layers, experts, top_k, expert_size, tokens, microbatches, fraction, tier, cap_experts, peers)
    (6, 12, 2, 1 << 20, 8, 2, 50, "PeerHBM", 20, 1),
    (6, 12, 2, 1 << 20, 8, 2, 100, "PeerHBM", 30, 3),
    (4, 60, 4, 17_301_504, 32, 2, 100, "PeerHBM", 40, 7),
    (4, 60, 4, 17_301_504, 32, 1, 75, "PeerHBM", 200, 2),
    (8, 16, 2, 157_286_400, 16, 2, 100, "PeerHBM", 9, 7),
    (5, 8, 2, 3 << 20, 4, 2, 25, "HostDRAM", 4, 1),
]


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("case", MOE_CASES, ids=[f"moe{i}" for i in range(len(MOE_CASES))])
def test_random_moe_placement_and_plan_match_reference(case, seed):
    """place_offloaded / rebalance residency (every handle key) and the serving
    tier + handle of every fetch of the decode, for fresh routing seeds,
    shapes, offload fractions, donor counts and capacities (some run out)."""
    import numpy as np
    mg = _golden_tools()
    from paper_2602_00328_b200 import moe as M
    from paper_2602_00328_b200.events import VirtualLoop
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.runtime import HarvestRuntime
    from tests.test_moe_parity import paper_h100_topology
    L, E, K, S, T, nmb, fraction, tier, cap_experts, peers = case
    ref_model = mg.moe.MoEProfile("diff", num_layers=L, num_experts=E, top_k=K, expert_size=S,
                                  compute_time_per_microbatch=1e-3)
    pipe = mg.moe.PipelineConfig(microbatch_tokens=T, num_microbatches=nmb)
    c = mg.fetch_plan(ref_model, pipe, fraction, mg.Tier(tier), cap_experts * S, peers, 100 + seed)
    model = M.MoEProfile("diff", L, E, K, S, 1e-3)
    active = [[tuple(x) for x in row] for row in c["active"]]
    trace = M.RoutingTrace(len(active), L, E, active, np.array(c["counts"], dtype=np.int64))
    topo, host_id = paper_h100_topology(peers, cap_experts * S)
    loop = VirtualLoop()
    rt = HarvestRuntime(loop, topo)
    res = M.ExpertResidency(model)
    M.place_offloaded(loop, rt, model, res, trace, fraction, Tier(tier), host_id)
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
    assert c["read_errors"] == 0


@pytest.mark.parametrize("seed", range(20))
def test_availability_timelines_match_reference(seed):
    """churn.markov_availability / availability_from_trace against the
    reference's traces.py:171-213 on fresh parameters: identical steps and
    identical level_at on a probe grid."""
    mg = _golden_tools()
    from paper_2602_00328_b200 import churn as C
    rng = random.Random(seed)
    n = rng.randint(1, 5)
    levels = [rng.randint(0, 1 << 34) for _ in range(n)]
    soj = [rng.choice([0.01, 0.05, 0.2, 1.0]) for _ in range(n)]
    horizon = rng.choice([0.5, 2.0, 10.0])
    want = mg.traces.markov_availability(levels, soj, seed, horizon)
    got = C.markov_availability(levels, soj, seed, horizon)
    assert [tuple(s) for s in got.steps] == [tuple(s) for s in want.steps]
    recs = [(rng.uniform(0, 100), rng.random()) for _ in range(rng.randint(1, 30))]
    cap = rng.choice([80 << 30, 180 << 30])
    res, head = rng.choice([0, 1 << 30]), rng.choice([0, 2 << 30])
    scale = rng.choice([1.0, 0.01])
    want2 = mg.traces.availability_from_trace(
        [mg.traces.SnapshotRecord("m", t, int(u * cap), cap) for t, u in recs], cap, scale, res, head)
    got2 = C.availability_from_trace([(t, int(u * cap) / cap) for t, u in recs], cap, scale, res, head)
    assert [tuple(s) for s in got2.steps] == [tuple(s) for s in want2.steps]
    for t in [x * horizon / 17 for x in range(18)]:
        assert got.level_at(t) == want.level_at(t)


@pytest.mark.parametrize("seed", range(10))
def test_calibrate_matches_reference(seed):
    """interconnect.calibrate / calibration_rms / transfer_time (interconnect.py:51-54,
    :168-221) on fresh noisy latency curves: the same fit to 1e-12 relative."""
    mg = _golden_tools()
    from harvestsim import interconnect as RI
    from paper_2602_00328_b200 import interconnect as I
    rng = random.Random(seed)
    fc, bw = rng.uniform(1e-6, 50e-6), rng.uniform(10e9, 900e9)
    pts = [(s, (fc + s / bw) * (1 + rng.uniform(-0.02, 0.02)))
           for s in sorted(rng.sample(range(4096, 64 << 20), rng.randint(2, 12)))]
    want = RI.calibrate(pts)
    got = I.calibrate(pts)
    assert got == pytest.approx(want, rel=1e-12)
    assert I.calibration_rms(pts, *got) == pytest.approx(RI.calibration_rms(pts, *want), rel=1e-12)
    link_r = RI.LinkSpec(RI.LinkKind.PEER_LINK, fc, bw, endpoints=(0, 1))
    link_o = I.LinkSpec(I.LinkKind.PEER_LINK, fc, bw, endpoints=(0, 1))
    for s in (1, 65536, 17_301_504):
        assert I.transfer_time(link_o, s) == RI.transfer_time(link_r, s)
