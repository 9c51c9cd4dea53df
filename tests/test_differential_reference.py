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
