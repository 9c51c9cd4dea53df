"""Shared definitions of the contract benchmark (bench.py): the workload, its routing, output."""
from __future__ import annotations

import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)



GiB = 1 << 30

METRIC = "expert-fetch GB/s"

from benchlib.workload import QWEN15, SEED, TOKENS  # noqa: E402
from benchlib.workload import routing as _routing  # noqa: E402

KV_TOKENS, KV_SLAB_BLOCKS = 131072, 64   # BASELINE configs[3]: one 128k-token Llama-3-8B sequence

def shape():
    """The workload shape (product-free; see benchlib/workload.py)."""
    layers = int(os.environ.get("HV_BENCH_QWEN_LAYERS", "0"))
    if layers:  # test-only: many ranks on one GPU (the reported config is the 24-layer model)
        from dataclasses import replace
        return replace(QWEN15, num_layers=layers)
    return QWEN15

def model():
    """The B200 arm's MoEProfile of the same shape."""
    from paper_2602_00328_b200.moe import MoEProfile
    w = shape()
    return MoEProfile(w.name, w.num_layers, w.num_experts, w.top_k, w.expert_size, hidden=w.hidden,
                      intermediate=w.intermediate)

def routing(m, steps, seed=SEED):
    return _routing(m, steps, seed, TOKENS)

def workload_config(m, n, source=None):
    """The workload both arms run (the same dict for the B200 arm and the
    reference arm at the same N): model shape, routing, fetched bytes per
    step and the N-GPU scenario.  Implementation details (source tier, fetch
    engine, pools) are reported outside `config`."""
    scenario = ("1 GPU: experts in the pinned host tier" if n <= 1 else
                f"{n} GPUs, one process each: every GPU a compute GPU whose experts sit in the HBM of "
                f"the N-1={n - 1} others")
    return {"workload": f"{m.name} expert fetch (BASELINE configs[1]): {m.num_layers} layers x "
                        f"{m.num_experts} experts x {m.expert_size} B, decode batch {TOKENS}, top-{m.top_k}, "
                        f"100% offloaded; one step = every layer's activated experts",
            "scenario": scenario,
            "l2": f"inputs larger than L2 (~{m.num_layers * 53 * m.expert_size / 1e9:.0f} GB fetched per step, "
                  "126 MB L2)",
            "routing": f"top-{m.top_k} of N(0,1) logits, seed {SEED}"}

def emit(line, a):
    s = json.dumps(line)
    print(s, flush=True)
    if a.out:
        with open(a.out, "a") as f:
            f.write(s + "\n")

def load_traffic():
    p = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}

def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return {"hbm_gbs": 6650.0, "fallback": "B200_PROFILING.md fallback 6.65 TB/s"}

def kv_slab_bytes():
    from paper_2602_00328_b200.kv import LLAMA3_8B
    return KV_SLAB_BLOCKS * LLAMA3_8B.block_bytes


def reference_checkers():
    """The reference's own event-log checkers (harvestsim/verify.py:25-88)
    from the unmodified install under baseline/_ref -- the bench's checker
    for release ordering under churn, never part of the measured path."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "harvestsim")):
        def unavailable(_log):
            return ["unchecked: baseline/_ref (the reference's verify.py) is not installed"]
        return unavailable, unavailable
    if ref not in sys.path:
        sys.path.append(ref)
    from harvestsim.verify import verify_no_runtime_writeback, verify_release_ordering
    return verify_release_ordering, verify_no_runtime_writeback
