"""Generate golden fixtures by running the REFERENCE (harvestsim) in this container.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Reads /root/reference/pkg/src (read-only; or HARVEST_REFERENCE).  The GPU
box only sees the committed JSON files.  On CPU,
tests/test_differential_reference.py also drives these runners against the
pip-installed copy under baseline/_ref (when present) on fresh random
scripts.  Every fixture records the reference file:line whose behaviour it
captures.
"""
from __future__ import annotations

import json
import os
import random
import sys
import zlib

sys.dont_write_bytecode = True
REF = os.environ.get("HARVEST_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from harvestsim import memalloc, moe, profiles, runtime, traces, verify  # noqa: E402
from harvestsim.events import Simulator  # noqa: E402
from harvestsim.interconnect import LinkKind, LinkSpec, Topology  # noqa: E402
from harvestsim.memalloc import DeviceSpec, Segment, Tier  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
GiB = 1 << 30


def dump(name, obj):
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, indent=None, separators=(",", ":"), sort_keys=True)
        f.write("\n")


def hkey(h):
    return None if h is None else [h.device_id, h.base, h.size, h.generation]


# ---------------------------------------------------------------- 1. identity
def gen_hashes():
    tags = []
    for model in ("qwen1.5-moe-a2.7b", "phi-3.5-moe", "qwen2-moe"):
        for layer in (0, 1, 23):
            for e in (0, 1, 59):
                tags.append(["expert", model, layer, e])
    for layer in (0, 31):
        for seq in (0, 3):
            for blk in (0, 255, 8191):
                tags.append(["kv", layer, seq, blk])
    tags += [["obj", i] for i in range(4)] + [["d", 0], ["b", 4096]]
    vals = [str(runtime.stable_hash64(*t)) for t in tags]
    exp = [str(moe.expert_content(moe.MOE_PROFILES["qwen2-moe"] if False else
                                  profiles.MOE_PROFILES["qwen2-moe"], 3, 7))]
    dump("stable_hash64.json", {"source": "runtime.py:38-44, moe.py:114-115",
                                "tags": tags, "values": vals,
                                "expert_content_qwen2_3_7": exp[0]})


# ---------------------------------------------------------------- 2. allocator
def gen_allocator():
    cases = []
    rng = random.Random(11)
    for case in range(40):
        usable = rng.choice([100, 1000, 1 << 20, 80 * GiB])
        st = memalloc.init_device(DeviceSpec(1, Tier.PEER_HBM, usable))
        ops, live = [], []
        for _ in range(rng.randint(20, 200)):
            if live and rng.random() < 0.45:
                seg = live.pop(rng.randrange(len(live)))
                memalloc.free_segment(st, seg)
                ops.append(["free", seg.base, seg.size, None])
            else:
                size = rng.randint(1, max(1, usable // rng.choice([3, 10, 50, 400])))
                seg = memalloc.alloc_best_fit(st, size)
                if seg is not None:
                    live.append(seg)
                ops.append(["alloc", size, None, None if seg is None else seg.base])
            memalloc.check_invariants(st)
        cases.append({"usable": usable, "ops": ops,
                      "free_list": [[s.base, s.size] for s in st.free_list],
                      "allocated_bytes": memalloc.allocated_bytes(st)})
    # SPEC.md:56-58 examples on hand-built free lists
    spec = []
    for fl, size in (([[0, 100], [200, 40]], 40), ([[0, 100], [200, 64], [300, 65]], 60), ([[0, 30]], 31)):
        st = memalloc.DeviceState(spec=DeviceSpec(1, Tier.PEER_HBM, 1000))
        st.free_list = [Segment(b, s) for b, s in fl]
        seg = memalloc.alloc_best_fit(st, size)
        spec.append({"free_list": fl, "size": size, "base": None if seg is None else seg.base,
                     "after": [[s.base, s.size] for s in st.free_list]})
    dump("allocator.json", {"source": "memalloc.py:74-138", "cases": cases, "spec_examples": spec})


# ---------------------------------------------------------------- 3. runtime decisions
def topo(peers, host_cap=64 * GiB, hops=None):
    devices = [DeviceSpec(0, Tier.LOCAL_HBM, 16 * GiB)]
    links = []
    hid = len(peers) + 1
    for i, (cap, reserved, headroom) in enumerate(peers, start=1):
        devices.append(DeviceSpec(i, Tier.PEER_HBM, cap, reserved=reserved, headroom=headroom))
        links.append(LinkSpec(LinkKind.PEER_LINK, 1e-6, 100e9, endpoints=(0, i),
                              hops=(hops or {}).get(i, 1)))
        links.append(LinkSpec(LinkKind.HOST_LINK, 10e-6, 10e9, endpoints=(i, hid)))
    devices.append(DeviceSpec(hid, Tier.HOST_DRAM, host_cap))
    links.append(LinkSpec(LinkKind.HOST_LINK, 10e-6, 10e9, endpoints=(0, hid)))
    return Topology(devices=devices, links=links)


LOG_KINDS = ("alloc", "alloc_nocapacity", "free_begin", "revoke_begin", "invalidate", "callback",
             "free", "reclaim", "availability_step", "transfer_start", "transfer_complete")


def log_of(sim):
    out = []
    for r in sim.log:
        if r.kind not in LOG_KINDS:
            continue
        d = {k: (list(v) if isinstance(v, tuple) else v) for k, v in r.data.items()
             if k in ("device", "base", "size", "gen", "reason", "cause", "client", "amount",
                      "revoked", "freed", "level", "src", "dst", "handle", "initiator")}
        out.append([r.kind, d])
    return out


def run_script(policy, peers, script, hops=None):
    """Replay a scripted op sequence on the reference; record every result."""
    sim = Simulator()
    rt = runtime.HarvestRuntime(sim, topo(peers, hops=hops), policy=policy)
    handles, results, cbs = {}, [], []
    for op in script:
        kind = op[0]
        if kind == "time":
            sim.run(until=op[1])
            results.append(None)
        elif kind == "alloc":
            _, name, size, pref, client = op
            h = rt.harvest_alloc(size, runtime.AllocationHints(preferred_devices=pref, client_id=client))
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
            except runtime.StaleHandleError:
                results.append("stale")
        elif kind == "revoke":
            rt.revoke(handles[op[1]], runtime.RevokeReason(op[2]))
            results.append("ok")
        elif kind == "touch":
            rt.touch(handles[op[1]])
            results.append("ok")
        elif kind == "reclaim":
            rev = rt.external_reclaim(op[1], op[2], order=op[3])
            results.append([hkey(h) for h in rev])
        elif kind == "availability":
            rt.apply_availability(op[1], [tuple(s) for s in op[2]])
            results.append("ok")
        elif kind == "read":  # app transfer peer -> local touching a handle
            h = handles[op[1]]
            if rt.is_live(h):
                rt.write_peer(h, ("t", op[1]), 1) if op[2] else None
                rt.app_transfer(src=(h.device_id, Segment(h.base, h.size)),
                                dst=(0, Segment(0, h.size)), size=h.size, tag=("t", op[1]), handle=h)
                results.append("issued")
            else:
                results.append("miss")
        elif kind == "run":
            sim.run()
            results.append(None)
        elif kind == "lookup":
            results.append(rt.is_live(handles[op[1]]))
        elif kind == "state":
            results.append({str(d): [rt.occupied_bytes(d), rt.harvestable(d)]
                            for d in rt.devices if rt.devices[d].spec.tier == Tier.PEER_HBM})
    sim.run()
    return {"results": results, "callbacks": cbs, "log": log_of(sim),
            "release_violations": verify.verify_release_ordering(sim.log),
            "writeback_violations": verify.verify_no_runtime_writeback(sim.log)}


def random_script(rng, n_ops, peers, with_time=True):
    script, names = [], []
    t = 0.0
    for i in range(n_ops):
        r = rng.random()
        if with_time and r < 0.1:
            t += rng.choice([0.0, 1e-6, 1e-3, 0.5, 3.0])
            script.append(["time", t])
        elif r < 0.5 or not names:
            name = f"h{i}"
            size = rng.choice([1 << 20, 3 << 20, 17_301_504, 64 << 10, rng.randint(1, 8 << 20)])
            pref = rng.choice([None, None, [rng.randint(1, len(peers))]])
            script.append(["alloc", name, size, pref, rng.choice(["moe", "kv", "default"])])
            names.append(name)
        elif r < 0.62:
            script.append(["free", rng.choice(names)])
        elif r < 0.74:
            script.append(["revoke", rng.choice(names), rng.choice(["Pressure", "Policy", "ExternalReclaim"])])
        elif r < 0.82:
            script.append(["read", rng.choice(names), True])
        elif r < 0.87:
            script.append(["touch", rng.choice(names)])
        elif r < 0.91:
            script.append(["reclaim", rng.randint(1, len(peers)), rng.choice([0, 1 << 20, 20 << 20, 1 << 40]),
                           rng.choice(["lru", "fifo"])])
        elif r < 0.95:
            script.append(["run"])
        else:
            script.append(["lookup", rng.choice(names)])
    script.append(["state"])
    return script


def gen_runtime():
    rng = random.Random(5)
    scenarios = []
    pol = runtime.Policy
    K = runtime.PolicyKind
    configs = [
        ("bestfit", pol(K.BEST_FIT), [(64 << 20, 0, 0), (40 << 20, 0, 0), (100 << 20, 8 << 20, 4 << 20)], None),
        ("locality", pol(K.LOCALITY), [(64 << 20, 0, 0), (64 << 20, 0, 0), (64 << 20, 0, 0)], {1: 2, 2: 1, 3: 3}),
        ("fairness", pol(K.FAIRNESS, fairness_budget_bytes_per_s=8 << 20, fairness_burst_bytes=24 << 20),
         [(128 << 20, 0, 0), (128 << 20, 0, 0)], None),
        ("stability", pol(K.STABILITY, stability_window_s=2.0, stability_max_revocations=2),
         [(64 << 20, 0, 0), (64 << 20, 0, 0), (64 << 20, 0, 0)], None),
    ]
    for name, p, peers, hops in configs:
        for seed in range(6):
            script = random_script(random.Random(zlib.crc32(f"{name}-{seed}".encode())), 120, peers)
            scenarios.append({"name": f"{name}-{seed}", "policy": p.kind.value,
                              "policy_params": [p.fairness_budget_bytes_per_s if p.fairness_budget_bytes_per_s != float("inf") else None,
                                                p.fairness_burst_bytes, p.stability_window_s,
                                                p.stability_max_revocations],
                              "peers": peers, "hops": hops, "script": script,
                              **run_script(p, peers, script, hops)})
    # two peers with 10 GiB and 2 GiB free, 1.5 GiB -> the 2 GiB peer
    spec_peers = [(10 * GiB, 0, 0), (2 * GiB, 0, 0)]
    s = [["alloc", "a", 3 * GiB // 2, None, "default"], ["state"]]
    scenarios.append({"name": "spec-bestfit-across-devices", "policy": "BestFit",
                      "policy_params": [None, None, 10.0, 3], "peers": spec_peers, "hops": None, "script": s,
                      **run_script(pol(), spec_peers, s)})
    # availability timeline driving reclaim (runtime.py:465-487)
    av_peers = [(64 << 20, 0, 0)]
    s = [["alloc", f"a{i}", 8 << 20, None, "moe"] for i in range(6)] + \
        [["touch", "a0"], ["time", 0.5], ["touch", "a3"],
         ["availability", 1, [[1.0, 40 << 20], [2.0, 10 << 20], [3.0, 64 << 20]]], ["run"], ["state"]]
    scenarios.append({"name": "availability-steps", "policy": "BestFit", "policy_params": [None, None, 10.0, 3],
                      "peers": av_peers, "hops": None, "script": s, **run_script(pol(), av_peers, s)})
    dump("runtime_scenarios.json", {"source": "runtime.py:119-487", "scenarios": scenarios})


# ---------------------------------------------------------------- 4. MoE fetch plan
QWEN15 = moe.MoEProfile("qwen1.5-moe-a2.7b", num_layers=24, num_experts=60, top_k=4,
                        expert_size=17_301_504, compute_time_per_microbatch=6.716e-3)
PHI35 = moe.MoEProfile("phi-3.5-moe", num_layers=32, num_experts=16, top_k=2,
                       expert_size=157_286_400, compute_time_per_microbatch=14.863e-3)


def fetch_plan(model, pipeline, fraction, tier, peer_capacity, num_peers, seed, skew=1.2):
    trace = moe.generate_routing(model, pipeline, skew, 0, seed)
    sim = Simulator()
    top = profiles.build_topology(profiles.PAPER_H100, num_peers=num_peers, peer_capacity=peer_capacity)
    rt = runtime.HarvestRuntime(sim, top)
    host_id = top.devices[-1].device_id
    res = moe.ExpertResidency(model)
    moe.place_offloaded(sim, rt, model, res, trace, fraction, tier, host_id)
    residency = {}
    for (layer, e), ent in res.entries.items():
        residency[f"{layer},{e}"] = [ent.tier.value, hkey(ent.handle)]
    n_setup = len(sim.log)
    metrics = moe.simulate_decode(sim, rt, model, pipeline, trace, res, host_id)
    stages = []
    cur = None
    for r in list(sim.log)[n_setup:]:
        if r.kind == "transfer_start" and r.data["dst"] == 0:
            tag = r.data["tag"]
            stages.append([tag[1], tag[2], "host" if r.data["src"] == host_id else "peer",
                           None if r.data["handle"] is None else list(r.data["handle"])])
    return {"active": [[list(a) for a in row] for row in trace.active],
            "counts": trace.counts.tolist(), "residency": residency, "fetches": stages,
            "reads": metrics.reads, "read_errors": metrics.read_errors,
            "tokens_per_s": metrics.tokens_per_s, "per_stage_advance_sum": sum(metrics.per_stage_advance)}


def gen_moe():
    out = {"source": "moe.py:73-111 (routing), :155-197 (rebalance), :282-313 (fetch hook), :354-383 (placement)"}
    p32 = moe.PipelineConfig(microbatch_tokens=32, num_microbatches=2)
    out["qwen15_b32_peer50"] = fetch_plan(QWEN15, p32, 50, Tier.PEER_HBM, 40 * QWEN15.expert_size, 1, 2)
    out["qwen15_b32_host100"] = fetch_plan(QWEN15, p32, 100, Tier.HOST_DRAM, 80 * GiB, 1, 2)
    out["qwen15_b32_peer100_7donors"] = fetch_plan(QWEN15, p32, 100, Tier.PEER_HBM, 180 * GiB, 7, 3)
    p16 = moe.PipelineConfig(microbatch_tokens=16, num_microbatches=2)
    out["phi35_b16_peer100_7donors"] = fetch_plan(PHI35, p16, 100, Tier.PEER_HBM, 11 * GiB, 7, 4)
    out["models"] = {m.name: [m.num_layers, m.num_experts, m.top_k, m.expert_size, m.compute_time_per_microbatch]
                     for m in (QWEN15, PHI35)}
    # the reference's own sweep numbers (profiles.py:89-104 models), for the record
    sweeps = {}
    for name in ("qwen2-moe", "phi-3.5-moe"):
        m = profiles.MOE_PROFILES[name]
        pc = moe.PipelineConfig(microbatch_tokens=64, num_microbatches=4)
        sweeps[name] = {t.value: [[r.fraction_pct, r.tokens_per_s] for r in
                                  moe.offload_sweep(m, pc, [0, 50, 100], t, 0)]
                        for t in (Tier.PEER_HBM, Tier.HOST_DRAM)}
    out["offload_sweep"] = sweeps
    dump("moe_fetch.json", out)


# ---------------------------------------------------------------- 5. traces
def gen_traces():
    GB = 1 << 30
    av = traces.markov_availability([0, 45 * GB, 90 * GB, 180 * GB], [0.05] * 4, seed=5, horizon=2.0)
    av2 = traces.markov_availability([10, 20], [10.0, 10.0], seed=1, horizon=100.0)
    dump("traces.json", {"source": "traces.py:190-213",
                         "markov_c5": av.steps, "markov_two_level": av2.steps})


if __name__ == "__main__":
    gen_hashes()
    gen_allocator()
    gen_runtime()
    gen_moe()
    gen_traces()
    print("golden fixtures written to", OUT)
