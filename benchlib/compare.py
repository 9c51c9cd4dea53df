"""Same-run comparisons (copy engine, latency curves, KV config-1 gather), engine probe and autotune."""
from __future__ import annotations

import json
import os
import statistics
import sys

import numpy as np

from benchlib.common import REPO, model


def measure_pcie_h2d(dev):
    import torch
    from paper_2602_00328_b200.pool import HostTier
    h = HostTier(1 << 30)
    d = torch.empty(1 << 30, dtype=torch.uint8, device=f"cuda:{dev}")
    s = torch.cuda.Stream(dev)
    best = 0.0
    with torch.cuda.stream(s):
        src = torch.from_numpy(h.view())
        for i in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            d.copy_(src, non_blocking=True)
            e1.record(s)
            e1.synchronize()
            if i:
                best = max(best, (1 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del src
    h.close()
    return best

def measure_peer_copy(dev, src_dev, nbytes=256 << 20):
    """Peer -> this GPU copy-engine rate (cudaMemcpyPeerAsync through torch's
    cross-device copy), best of 5, GB/s; None when the donor is this GPU (a
    single-GPU stand-in) or the copy fails."""
    import torch
    if src_dev == dev:
        return None
    try:
        src = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{src_dev}")
        d = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dev}")
        s = torch.cuda.Stream(dev)
        best = 0.0
        with torch.cuda.stream(s):
            for i in range(6):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                d.copy_(src, non_blocking=True)
                e1.record(s)
                e1.synchronize()
                if i:
                    best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        del src, d
        return best or None
    except Exception:   # noqa: BLE001 -- the fallback peak is reported instead
        return None


PROBE_CHILD = r"""
import json, sys
sys.path.insert(0, {repo!r})
import torch
from paper_2602_00328_b200 import fetch as F
from paper_2602_00328_b200.pool import PeerPool, RemotePool
if {mode!r} == "remote":
    p = RemotePool({path!r}, {donor}, {chunk}, {chunk}, {dev})
    p.commit(0, {chunk})
    va = p.va
else:
    p = PeerPool.import_ipc(bytes.fromhex({handle!r}), {donor}, {nbytes}, {dev})
    va = p.va
n = min(4 << 20, {chunk})
a = torch.empty(n, dtype=torch.uint8, device="cuda:{dev}")
b = torch.empty(n, dtype=torch.uint8, device="cuda:{dev}")
src = F.ptrs_tensor([va], "cuda:{dev}")
sz = F.ptrs_tensor([n], "cuda:{dev}")
if {mode!r} == "remote":   # a fresh chunk of its own: give it content (the IPC slab is only read)
    F.fill_content(src, sz, [7])
F.batch_copy(src, F.ptrs_tensor([a.data_ptr()], "cuda:{dev}"), sz, engine="ldg")
F.batch_copy(src, F.ptrs_tensor([b.data_ptr()], "cuda:{dev}"), sz, engine={engine!r})
torch.cuda.synchronize()
print(json.dumps({{"ok": bool(torch.equal(a, b))}}))
p.close()
"""

def probe_engines_on_peer(node, donor_rank: int, donor_dev: int, dev: int) -> dict:
    """Run each non-LDG engine on a real peer pointer in a throw-away child
    process: a fault there cannot poison this process's CUDA context.  The
    child maps one chunk of the donor through the node's pool mechanism
    (a RemotePool connection to the donor's server, or the IPC slab)."""
    import subprocess
    from paper_2602_00328_b200.pool import _socket_path
    # the LDG family issues the same LDG.E.128 loads (hint / unroll differ):
    # only the bulk-copy (TMA) engine is proven out of process
    ok = {"ldg": True, "ldg256": True, "ldg16": True}
    remote = node.mode == "remote"
    try:
        own = node._readers[node.layout.donors_of(node.rank).index(donor_rank)]
    except (IndexError, ValueError):
        return {**ok, "tma": False}
    for engine in ("tma",):
        try:   # any failure here (even building the child's script) only rules the engine out
            code = PROBE_CHILD.format(repo=REPO, mode=node.mode, path=_socket_path("main", donor_rank),
                                      handle="" if remote else node.ipc_handles[donor_rank].hex(),
                                      donor=donor_dev, nbytes=node.layout.slab_bytes(donor_rank),
                                      chunk=getattr(own, "chunk_bytes", 32 << 20) if remote else 4 << 20,
                                      dev=dev, engine=engine)
            r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=180)
            ok[engine] = r.returncode == 0 and '"ok": true' in r.stdout
        except Exception:
            ok[engine] = False
    return ok

def autotune(layer_desc, stream, stream_h, F, reps=3, engines=("ldg", "ldg256", "ldg16", "tma", "ce", "auto"),
             barrier=None, max_over_ranks=None, checked=None):
    """Time one layer's real fetch (host descriptor arrays, the product's
    hv_swap_blocks_batch entry point) under each engine x grid cap; pick the
    fastest.  "ce" is the copy engine (cudaMemcpyAsync per contiguous run), "auto" the
    library's engine per source (copy engine for large host-tier objects,
    kernel otherwise).  Multi-rank: every rank times the same candidate at the
    same moment (barrier before each), so the measurement includes the
    contention of all readers on the donors' links; a candidate's time is the
    max over ranks.  ``checked=(scratch, errors)``: time the fetch with its
    fused content check (hv_swap_blocks_batch_checked), the product's peer
    path."""
    import torch
    from paper_2602_00328_b200 import _native as N
    sp, dp, sz, nb = layer_desc[:4]
    rows = []

    def launch(engine, max_ctas):
        if checked is None:
            F.swap_blocks_batch(sp, dp, sz, engine=engine, max_ctas=max_ctas, stream=stream_h)
        else:
            ex = layer_desc[4]
            N.call("hv_swap_blocks_batch_checked", sp.ctypes.data, dp.ctypes.data, sz.ctypes.data, ex.ctypes.data,
                   len(sp), N.ENGINES[engine], max_ctas, checked[0].data_ptr(), 0, checked[1].data_ptr(), stream_h)

    for engine in engines:
        grids = (0,) if engine.split("+")[0] in ("ce", "auto") else (0, 296, 148)
        for max_ctas in grids:
            launch(engine, max_ctas)  # warm
            stream.synchronize()
            if barrier is not None:
                barrier()
            ts = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                launch(engine, max_ctas)
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
            t = statistics.median(ts)
            if max_over_ranks is not None:
                t = max_over_ranks(t)
            rows.append({"engine": engine, "max_ctas": max_ctas, "GBps": nb / t / 1e9})
    best = max(rows, key=lambda r: r["GBps"])
    return {"best": best, "candidates": rows}

def same_run_comparisons(dev, m, a, source, fetcher=None, n=53):
    """Same-box comparisons for one layer's worth of experts (n x 17.3 MB):
    the copy-engine paths on the same source (cudaMemcpyAsync: the
    paper's/vLLM's data path) and the same kernel on a local-HBM source
    against the HBM roofline (kernel quality independent of the link)."""
    import torch
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.pool import HostTier
    S = m.expert_size
    dst = torch.empty(n * S, dtype=torch.uint8, device=f"cuda:{dev}")
    loc = torch.empty(n * S, dtype=torch.uint8, device=f"cuda:{dev}")
    s = torch.cuda.Stream(dev)

    def t(fn, iters=5):
        best = []
        for i in range(iters + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            if i >= 2:
                best.append(e0.elapsed_time(e1) * 1e-3)
        return statistics.median(best)

    def pct(fn, iters=100):
        """p50/p99 of one fetch's device time over `iters` launches (after 5 warmups)."""
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        for _ in range(5):
            fn()
        for e0, e1 in evs:
            e0.record(s)
            fn()
            e1.record(s)
        s.synchronize()
        us = np.array([e0.elapsed_time(e1) * 1e3 for e0, e1 in evs])
        return {"p50": float(np.percentile(us, 50)), "p99": float(np.percentile(us, 99)), "n": iters}

    out = {}
    dp = F.ptrs_tensor([dst.data_ptr() + i * S for i in range(n)], f"cuda:{dev}")
    sz = F.ptrs_tensor([S] * n, f"cuda:{dev}")
    lp = F.ptrs_tensor([loc.data_ptr() + i * S for i in range(n)], f"cuda:{dev}")
    keng = getattr(a, "kernel_engine", a.engine)   # the SM kernel engine (device-array entry points)
    dt = t(lambda: F.batch_copy(lp, dp, sz, engine=keng, stream=s.cuda_stream))
    hbm_peak = 6553.0
    try:
        hbm_peak = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    out["roofline_local_source"] = {"bound": "hbm", "achieved": 2 * n * S / dt / 1e9, "peak": hbm_peak,
                                    "unit": "GB/s", "frac": 2 * n * S / dt / 1e9 / hbm_peak,
                                    "note": "same K2 kernel, local-HBM source: read+write bytes / time vs "
                                            "MEASURED_PEAKS.json hbm_gbs (copy, read+write)"}
    hd = np.array([dst.data_ptr() + i * S for i in range(n)], dtype=np.uint64)
    hz = np.full(n, S, dtype=np.uint64)
    h = HostTier(n * S)
    hs = np.array([h.host_address(i * S) for i in range(n)], dtype=np.uint64)
    lat = {}
    lat["kernel_host"] = t(lambda: F.batch_copy(F.ptrs_tensor([h.device_address(0)], f"cuda:{dev}"), dp[:1],
                                                sz[:1], engine=keng, stream=s.cuda_stream)) * 1e6
    hda = np.array([h.device_address(0)], dtype=np.uint64)
    lat["product_host"] = t(lambda: F.swap_blocks_batch(hda, hd[:1], hz[:1], engine=a.engine,
                                                        stream=s.cuda_stream)) * 1e6
    lat["product_engine"] = a.engine
    lat["copy_engine_host"] = t(lambda: F.ce_batch_copy(hs[:1], hd[:1], hz[:1], batched=False,
                                                        stream=s.cuda_stream)) * 1e6
    if source == "host":
        dce = t(lambda: F.ce_batch_copy(hs, hd, hz, batched=True, stream=s.cuda_stream))
        out["copy_engine_same_source_GBps"] = n * S / dce / 1e9
    else:
        # peer experts of layer 0 (spread over every donor)
        ps = np.ascontiguousarray(fetcher.src_addr[0, :n])
        pdev = F.ptrs_tensor(ps, f"cuda:{dev}")
        dce = t(lambda: F.ce_batch_copy(ps, hd, hz, batched=True, stream=s.cuda_stream))
        out["copy_engine_same_source_GBps"] = n * S / dce / 1e9
        dce_loop = t(lambda: F.ce_batch_copy(ps, hd, hz, batched=False, stream=s.cuda_stream))
        out["copy_engine_peer_per_object_GBps"] = n * S / dce_loop / 1e9
        lat["kernel_peer"] = t(lambda: F.batch_copy(pdev[:1], dp[:1], sz[:1], engine=keng,
                                                    stream=s.cuda_stream)) * 1e6
        lat["copy_engine_peer"] = t(lambda: F.ce_batch_copy(ps[:1], hd[:1], hz[:1], batched=False,
                                                            stream=s.cuda_stream)) * 1e6
        # the host figure is the faster of the two host paths (copy engine or kernel)
        lat["peer_vs_host_speedup"] = min(lat["copy_engine_host"], lat["product_host"]) / lat["kernel_peer"]
    # latency distribution (p50/p99 over >= 100 iterations)
    dist_us = {"kernel_host": pct(lambda: F.batch_copy(F.ptrs_tensor([h.device_address(0)], f"cuda:{dev}"), dp[:1],
                                                       sz[:1], engine=keng, stream=s.cuda_stream)),
               "product_host": pct(lambda: F.swap_blocks_batch(hda, hd[:1], hz[:1], engine=a.engine,
                                                               stream=s.cuda_stream))}
    if source == "peer":
        dist_us["kernel_peer"] = pct(lambda: F.batch_copy(pdev[:1], dp[:1], sz[:1], engine=keng,
                                                          stream=s.cuda_stream))
    lat["distribution_us"] = dist_us
    out["single_expert_latency_us"] = lat
    # KV config 1 (BASELINE configs[0] shape): 1,024 x 64 KiB pages = one layer
    # of 4 sequences x 4k tokens, gathered by K1 from the tier under test
    page, npg = 65536, 1024
    rng = np.random.default_rng(5)
    kv = {}
    kdst = torch.empty(npg * page, dtype=torch.uint8, device=f"cuda:{dev}")
    hp = HostTier(4 * npg * page)
    host_pages = F.ptrs_tensor([hp.device_address(int(p) * page) for p in rng.permutation(4 * npg)[:npg]],
                               f"cuda:{dev}")
    dt_h = t(lambda: F.kv_gather(host_pages, page, dst=kdst, engine=keng, stream=s.cuda_stream))
    kv["host_us"], kv["host_GBps"] = dt_h * 1e6, npg * page / dt_h / 1e9
    kv["distribution_us"] = {"host": pct(lambda: F.kv_gather(host_pages, page, dst=kdst, engine=keng,
                                                              stream=s.cuda_stream))}
    if source == "peer":
        base = fetcher.src_addr[0, :n]   # peer memory of n experts viewed as page slots
        slots = [int(base[i]) + j * page for i in range(n) for j in range(S // page)]
        peer_pages = F.ptrs_tensor([slots[int(p)] for p in rng.permutation(len(slots))[:npg]], f"cuda:{dev}")
        dt_p = t(lambda: F.kv_gather(peer_pages, page, dst=kdst, engine=keng, stream=s.cuda_stream))
        kv["peer_us"], kv["peer_GBps"] = dt_p * 1e6, npg * page / dt_p / 1e9
        kv["peer_vs_host_speedup"] = dt_h / dt_p
        kv["distribution_us"]["peer"] = pct(lambda: F.kv_gather(peer_pages, page, dst=kdst, engine=keng,
                                                                 stream=s.cuda_stream))
    out["kv_config1_layer_gather"] = kv
    out.update(latency_curves(dev, a, s, t, h, fetcher if source == "peer" else None))
    try:
        out["kv_fallback_measured"] = kv_fallback_measured(dev, h)
    except Exception as e:   # reported, never fatal
        out["kv_fallback_measured"] = {"error": repr(e)[:300]}
    hp.close()
    h.close()
    return out

def latency_curves(dev, a, s, t, host, fetcher):
    """Measured single-object fetch latency vs size on each available tier,
    refit with the reference's own calibrate() (interconnect.py:168-200), and
    the paper's KV reload-latency experiment (Fig 7:
    FP16 KV, 100..8000 entries, host vs peer) measured instead of modeled."""
    import torch
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.interconnect import CalibrationError, calibrate, calibration_rms
    sizes = [65536, 262144, 1 << 20, 4 << 20, 17_301_504]
    dst = torch.empty(max(sizes) + (8000 * 70_272), dtype=torch.uint8, device=f"cuda:{dev}")
    tiers = {"host": host.device_address(0)}
    if fetcher is not None:
        tiers["peer"] = int(fetcher.src_addr[0, 0])
    one = F.ptrs_tensor([S for S in [0]], f"cuda:{dev}")
    curves, fits = {}, {}
    hdst = np.array([dst.data_ptr()], dtype=np.uint64)
    for name, base in tiers.items():
        pts = []
        for nb in sizes:
            sp = np.array([base], dtype=np.uint64)
            sz = np.array([nb], dtype=np.uint64)
            # the product's fetch entry point and engine (per source under "auto")
            pts.append((nb, t(lambda: F.swap_blocks_batch(sp, hdst, sz, engine=a.engine, stream=s.cuda_stream))))
        curves[name] = [[nb, lat * 1e6] for nb, lat in pts]
        try:
            fc, bw = calibrate(pts)
            fits[name] = {"fixed_cost_us": fc * 1e6, "bandwidth_GBps": bw / 1e9,
                          "rms_rel": calibration_rms(pts, fc, bw)}
        except CalibrationError as e:   # a noisy curve (e.g. under a profiler) must not cost the bench line
            fits[name] = {"error": str(e)}
    out = {"latency_vs_size_us": curves, "calibrated_links": fits}
    if fetcher is not None:
        rows = []
        for model, bpe in (("kimi-k2", 70_272), ("mistral-large-3", 12_800)):   # profiles.py:116-122
            for e in (100, 500, 1000, 2000, 4000, 8000):
                nb = e * bpe
                lat = {}
                for name, base in tiers.items():
                    sp = np.array([base], dtype=np.uint64)
                    sz = np.array([nb], dtype=np.uint64)
                    lat[name] = t(lambda: F.swap_blocks_batch(sp, hdst, sz, engine=a.engine, stream=s.cuda_stream))
                rows.append([model, e, lat["host"] * 1e6, lat["peer"] * 1e6, lat["host"] / lat["peer"]])
        out["kv_reload_latency_experiment"] = {"columns": ["model", "entries", "host_us", "peer_us", "speedup"],
                                               "rows": rows,
                                               "paper_h100": "kimi-k2 5.42x@100 -> 5.68x@8000 (PAPER.md:319)"}
    del one
    return out


def kv_fallback_measured(dev, host):
    """§8(f)4: resolve_fallback on B200-measured costs --
    the host link refit with calibrate() from real fetch latencies, and the
    Llama-3-8B recompute cost (chunked prefill through all 32 layers) -- with
    the decision boundary solved for both the SPEC's linear rate and the
    measured curve."""
    from paper_2602_00328_b200.costs import LLAMA3_8B_DENSE, fallback_crossover, measure_host_link, measure_recompute
    from paper_2602_00328_b200.kv import LLAMA3_8B
    link, fit = measure_host_link(host, dev)
    curve = measure_recompute(LLAMA3_8B_DENSE, chunks=(16, 64, 256, 1024, 4096), device=dev)
    bpe = LLAMA3_8B.bytes_per_entry
    rate = curve.per_entry_rate
    return {"model": LLAMA3_8B.name, "bytes_per_entry": bpe, "host_link": fit,
            "recompute_prefill_us": [[e, t * 1e6] for e, t in curve.points],
            "recompute_us_per_entry_large_chunk": rate * 1e6,
            "host_fetch_us_per_entry": bpe / link.bandwidth * 1e6,
            "crossover_linear_rate": fallback_crossover(link, bpe, rate),
            "crossover_measured_curve": fallback_crossover(link, bpe, curve),
            "note": "recompute = prefill of the block's tokens through every layer (attention over the chunk "
                    "only: a lower bound); FetchFromHost iff host transfer_time <= recompute time"}
