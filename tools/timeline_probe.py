"""Device timeline of the fetch / compute overlap, recorded by CUPTI (the
torch.profiler / Kineto activity trace: every kernel and copy-engine transfer
with its stream and device timestamps), independent of the decoders' own
CUDA events.  nsys is not in this image; this is the same kind of record.

Scenarios (one GPU; the "peer" tier is a self-donor VMM pool, i.e. HBM), each
a decode step captured as a CUDA graph and replayed (eager steps under a
profiler are host-launch-bound and show the CPU, not the device):
  moe_peer_staged    Qwen 8-layer slice, every expert in the peer pool, staged
                     decode with 2 micro-batches: K2 fetch on the fetch stream
                     (64 CTAs), router + expert FFN on the compute stream
  moe_host_staged    the same experts in the pinned host tier, K2 over PCIe
                     (the graph-capturable device-side plan)
  kv_peer_gather     Llama-3-8B config 1 (4 x 4k): K1 page gather on the KV
                     stream, K5 attention on the compute stream
  kv_peer_in_place   the same, K5 reading the peer pages in place (programmatic
                     dependent launch across layers)

For each: intervals of the fetch class (K1/K2 kernels, H2D copies) and of the
compute class (everything else) are merged per class and intersected:
`fetch_hidden_frac` = share of fetch time during which a compute kernel also
ran, `compute_hidden_frac` the converse, `fetch_utilization` = fetch time /
span (1.0 = the link never idles in a fetch-bound step).  Writes
<out>/<tag>_timeline.json and the raw traces (gzip) next to it.

    python tools/timeline_probe.py [--tag r2] [--out-dir gpurun_out]
"""
import argparse
import gzip
import json
import os
import shutil
import sys
import tempfile

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

FETCH_KERNELS = ("CopyOp", "page_copy", "block_copy", "upload_desc")


def _merge(iv):
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def _length(iv):
    return sum(b - a for a, b in iv)


def _intersect(x, y):
    i = j = 0
    out = []
    while i < len(x) and j < len(y):
        a, b = max(x[i][0], y[j][0]), min(x[i][1], y[j][1])
        if a < b:
            out.append([a, b])
        if x[i][1] < y[j][1]:
            i += 1
        else:
            j += 1
    return out


def analyse(trace_path):
    opener = gzip.open if trace_path.endswith(".gz") else open
    ev = json.load(opener(trace_path))["traceEvents"]
    dev = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    fetch, comp, streams = [], [], {}
    for e in dev:
        iv = (float(e["ts"]), float(e["ts"]) + float(e["dur"]))
        name = e.get("name", "")
        is_fetch = (e["cat"] == "gpu_memcpy" and "HtoD" in name) or any(k in name for k in FETCH_KERNELS)
        (fetch if is_fetch else comp).append(iv)
        s = (e.get("args") or {}).get("stream")
        st = streams.setdefault(str(s), {"events": 0, "busy_us": 0.0, "fetch_events": 0})
        st["events"] += 1
        st["busy_us"] += float(e["dur"])
        st["fetch_events"] += int(is_fetch)
    f, c = _merge(fetch), _merge(comp)
    both = _intersect(f, c)
    span = (max(b for _, b in f + c) - min(a for a, _ in f + c)) if f or c else 0.0
    return {"events": len(dev), "fetch_events": len(fetch), "compute_events": len(comp),
            "fetch_busy_us": _length(f), "compute_busy_us": _length(c), "overlap_us": _length(both),
            "span_us": span,
            "fetch_hidden_frac": _length(both) / _length(f) if f else None,
            "compute_hidden_frac": _length(both) / _length(c) if c else None,
            "fetch_utilization": _length(f) / span if span else None,
            # > 1 when kernels of the same class overlap each other (e.g. K5 of
            # layer l+1 starting while layer l drains, programmatic dependent launch)
            "compute_concurrency": sum(b - a for a, b in comp) / _length(c) if c else None,
            "streams": streams}


def profiled(fn, steps, path):
    from torch.profiler import ProfilerActivity, profile
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            fn()
        torch.cuda.synchronize()
    prof.export_chrome_trace(path)
    return analyse(path)


def moe_case(kind, tmp):
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.moe import (ExpertFetcher, ExpertResidency, ExpertStore, MoEProfile, RoutingTrace,
                                           place_offloaded)
    from paper_2602_00328_b200.system import HarvestSystem
    from benchlib.workload import QWEN15
    import numpy as np
    m = MoEProfile(QWEN15.name, 8, QWEN15.num_experts, QWEN15.top_k, QWEN15.expert_size, hidden=QWEN15.hidden,
                   intermediate=QWEN15.intermediate)
    nbytes = m.num_layers * m.num_experts * m.expert_size
    peer = kind == "moe_peer_staged"
    sysm = HarvestSystem(0, donors=[0] if peer else [], donor_bytes=nbytes + (64 << 20), host_bytes=nbytes,
                         local_bytes=1, log_transfers=False)
    try:
        store = ExpertStore(m, sysm.host_id, sysm.host)
        store.fill_host(0, weights=True)
        residency = ExpertResidency(m)
        if peer:
            trace = RoutingTrace(1, m.num_layers, m.num_experts, [],
                                 np.ones((m.num_layers, m.num_experts), dtype=np.int64))
            place_offloaded(sysm.loop, sysm.runtime, m, residency, trace, 100, Tier.PEER_HBM, sysm.host_id,
                            store=store)
            sysm.loop.run()
            n_peer = sum(1 for ent in residency.entries.values() if ent.tier == Tier.PEER_HBM)
        else:
            n_peer = 0
        f = ExpertFetcher(sysm.runtime, m, residency, store)
        dec = MoEDecoder(f, tokens=32, microbatches=2, seed=0, max_ctas=64 if peer else 0)
        dec.capture_graph()
        path = os.path.join(tmp, f"{kind}.json")
        rep = profiled(lambda: dec.step(dec.x0), 3, path)
        rep.update({"layers": m.num_layers, "experts_in_peer_pool": n_peer, "tokens": 32, "microbatches": 2,
                    "fetch_max_ctas": 64 if peer else 0, "steps": 3, "cuda_graph": True})
        del dec
        torch.cuda.synchronize()
        sysm.loop.run()
        return rep, path
    finally:
        sysm.close()


def kv_case(tmp, fused):
    from paper_2602_00328_b200.kv import LLAMA3_8B, KVCacheManager
    from paper_2602_00328_b200.kv_decode import KVAttentionDecoder
    from paper_2602_00328_b200.runtime import Durability
    from paper_2602_00328_b200.system import HarvestSystem
    m = LLAMA3_8B
    batch, ctx = 4, 4096
    nblk = batch * ctx // m.block_tokens
    sysm = HarvestSystem(0, donors=[0], donor_bytes=(nblk // 64 + 2) * 64 * m.block_bytes, host_bytes=1,
                         local_bytes=1)
    try:
        kv = KVCacheManager(sysm, m, local_blocks=nblk, host_blocks=1, slab_blocks=64,
                            durability=Durability.LOSSY, content="fp16")
        for s in range(batch):
            kv.append_kv(s, ctx)
        kv.evict(nblk * m.block_bytes)
        dec = KVAttentionDecoder(kv, list(range(batch)), q_heads=32, seed=1, fused=fused)
        dec.capture_graph()
        name = "kv_peer_in_place" if fused else "kv_peer_gather"
        path = os.path.join(tmp, f"{name}.json")
        rep = profiled(dec.step, 3, path)
        rep.update({"config": "config 1: 4 x 4k tokens, 32 layers, KV pages in the peer pool, "
                              + ("K5 in place" if fused else "gather mode (K1 then K5)"),
                    "steps": 3, "cuda_graph": True})
        del dec
        torch.cuda.synchronize()
        sysm.loop.run()
        kv.close()
        return rep, path
    finally:
        sysm.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r2")
    ap.add_argument("--out-dir", default=os.path.join(REPO, "gpurun_out"))
    a = ap.parse_args()
    os.makedirs(a.out_dir, exist_ok=True)
    tmp = tempfile.mkdtemp()
    out = {"source": "torch.profiler (Kineto/CUPTI activity trace: device timestamps of every kernel and copy)",
           "note": "one GPU; the peer tier is a self-donor VMM pool (HBM), so these show the overlap "
                   "structure, not NVLink rates"}
    for name, fn in (("moe_peer_staged", lambda: moe_case("moe_peer_staged", tmp)),
                     ("moe_host_staged", lambda: moe_case("moe_host_staged", tmp)),
                     ("kv_peer_gather", lambda: kv_case(tmp, False)),
                     ("kv_peer_in_place", lambda: kv_case(tmp, True))):
        try:
            rep, path = fn()
            with open(path, "rb") as src, gzip.open(os.path.join(a.out_dir, f"{a.tag}_timeline_{name}.json.gz"),
                                                    "wb") as dst:
                shutil.copyfileobj(src, dst)
            out[name] = rep
        except Exception as e:  # report the scenario, keep the others
            out[name] = {"error": repr(e)[:400]}
        print(name, json.dumps({k: v for k, v in out[name].items() if k != "streams"}), flush=True)
    with open(os.path.join(a.out_dir, f"{a.tag}_timeline.json"), "w") as fo:
        json.dump(out, fo, indent=1)


if __name__ == "__main__":
    main()
