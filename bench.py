#!/usr/bin/env python
"""Harvest-on-B200 contract benchmark: expert fetch GB/s (BASELINE.json configs[1]).

Workload (config 2): Qwen1.5-MoE-A2.7B-shaped experts (24 layers x 60 experts,
17,301,504 B each, bf16 gate+up+down), decode batch 32, top-4 routing over
N(0,1) router logits, 100% of experts offloaded.  One step = one decode step:
for each of the 24 layers, the distinct activated experts (~53) are fetched
into local HBM with ONE launch of the K2 batched-fetch kernel (~22 GB/step).

* N=1 (one GPU): experts live in the pinned host tier (the authoritative copy);
  the fetch reads them over PCIe ("1 GPU (host tier only)").
* N>1 (torchrun, one process per GPU): every rank is a compute GPU whose
  experts were placed by its own HarvestRuntime (harvest_alloc, best-fit) in the
  donated HBM of the N-1 other GPUs (cudaIpc pools); the fetch pulls them over
  NVLink 5 / NVSwitch.  No collective on the data path ("scaling": "weak").

``value``: device-resident descriptors, the timed region holds only the fetch
launches.  ``e2e``: the same steps through the public fetch hook
(ExpertFetcher.issue_fetches: host routing -> descriptors staged H2D -> launch)
plus a per-step verification kernel whose mismatch counts are read back D2H.

``--impl reference``: the reference CPU path (oracle port of the fetch, a
memcpy gather from the host-authoritative copy) on the box's host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

GiB = 1 << 30
METRIC = "peer-fetch GB/s"
TOKENS, SEED = 32, 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--engine", default="auto", choices=["auto", "ldg", "ldg256", "tma"])
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--cpu-baseline-s", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--no-kv", action="store_true", help="skip the config-4 long-context KV measurement")
    ap.add_argument("--no-phi", action="store_true", help="N>1: skip the config-3 Phi-3.5-MoE decode phase")
    ap.add_argument("--no-churn", action="store_true", help="skip the config-5 churn phase")
    ap.add_argument("--phi-layers", type=int, default=32,
                    help="layers of the Phi-3.5-MoE phase (32 = the real model; fewer only for single-GPU tests)")
    ap.add_argument("--overlap-max-ctas", type=int, default=64,
                    help="fetch grid cap in the 2-micro-batch (overlapped) decode")
    ap.add_argument("--no-host-compare", action="store_true",
                    help="N>1: skip rank 0's host-offload decode comparison")
    a = ap.parse_args()
    a.warmup = max(3, a.warmup)
    return a


def model():
    from paper_2602_00328_b200.moe import QWEN15_MOE_A27B, MoEProfile
    layers = int(os.environ.get("HV_BENCH_QWEN_LAYERS", "0"))
    if layers:  # test-only: many ranks on one GPU (the reported config is the 24-layer model)
        m = QWEN15_MOE_A27B
        return MoEProfile(m.name, layers, m.num_experts, m.top_k, m.expert_size, hidden=m.hidden,
                          intermediate=m.intermediate)
    return QWEN15_MOE_A27B


def routing(m, steps, seed=SEED):
    from paper_2602_00328_b200.moe import topk_routing
    return topk_routing(m, TOKENS, steps, seed)


def workload_config(m, n, source):
    return {"workload": f"{m.name} expert fetch (BASELINE configs[1]): {m.num_layers} layers x "
                        f"{m.num_experts} experts x {m.expert_size} B, decode batch {TOKENS}, top-{m.top_k}, "
                        f"100% offloaded; one step = every layer's activated experts",
            "source_tier": source, "donors_per_rank": max(0, n - 1),
            "l2": f"inputs larger than L2 (~{m.num_layers * 53 * m.expert_size / 1e9:.0f} GB fetched per step, "
                  "126 MB L2)",
            "routing": f"top-{m.top_k} of N(0,1) logits, seed {SEED}"}


# --------------------------------------------------------------------- CPU paths
def cpu_gather_sample(m, host_buf, route_steps, seconds, threads):
    """Oracle port of the fetch (memcpy gather of the activated experts from
    the host-authoritative copy) on host cores, for ~``seconds``."""
    from oracle import harvest_oracle as O
    dst = np.empty(m.num_experts * m.expert_size, dtype=np.uint8)
    base = host_buf.ctypes.data if isinstance(host_buf, np.ndarray) else host_buf
    moved, t0, layers = 0, time.perf_counter(), 0
    while True:
        for step in route_steps:
            for layer, ex in enumerate(step):
                src = [base + ((layer * m.num_experts + int(e)) % (host_nexp(m, host_buf))) * m.expert_size for e in ex]
                dp = [dst.ctypes.data + i * m.expert_size for i in range(len(ex))]
                O.gather(src, dp, [m.expert_size] * len(ex), threads=threads)
                moved += len(ex) * m.expert_size
                layers += 1
                if time.perf_counter() - t0 >= seconds:
                    dt = time.perf_counter() - t0
                    return moved / dt / 1e9, dt, layers, moved


def host_nexp(m, host_buf):
    return (host_buf.size // m.expert_size) if isinstance(host_buf, np.ndarray) else m.num_layers * m.num_experts


def cpu_host_copy(m, n_experts):
    """A host-resident expert table for the CPU legs (content from the oracle)."""
    from oracle import harvest_oracle as O
    from paper_2602_00328_b200.runtime import stable_hash64
    buf = np.empty(n_experts * m.expert_size, dtype=np.uint8)
    O.fill_batch([buf.ctypes.data + i * m.expert_size for i in range(n_experts)], [m.expert_size] * n_experts,
                 [stable_hash64("expert", m.name, i // m.num_experts, i % m.num_experts) for i in range(n_experts)],
                 threads=os.cpu_count() or 1)
    return buf


def run_reference(a):
    """--impl reference: the oracle port timed on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    m = model()
    threads = os.cpu_count() or 1
    sample_experts = 4 * m.num_experts          # 4 layers' worth of distinct experts (4.15 GB)
    host = cpu_host_copy(m, sample_experts)
    routes = routing(m, a.steps + a.warmup)
    per_step = []

    def one_step(step):
        # bounded sample of the step: its first 4 layers (the same activated sets)
        from oracle import harvest_oracle as O
        dst = one_step.dst
        moved = 0
        t0 = time.perf_counter()
        for layer in range(4):
            ex = step[layer]
            src = [host.ctypes.data + (layer * m.num_experts + int(e)) * m.expert_size for e in ex]
            dp = [dst.ctypes.data + i * m.expert_size for i in range(len(ex))]
            O.gather(src, dp, [m.expert_size] * len(ex), threads=threads)
            moved += len(ex) * m.expert_size
        return moved, time.perf_counter() - t0

    one_step.dst = np.empty(m.num_experts * m.expert_size, dtype=np.uint8)
    for s in range(a.warmup):
        one_step(routes[s])
    moved = dt = 0.0
    for s in range(a.warmup, a.warmup + a.steps):
        mv, t = one_step(routes[s])
        moved += mv
        dt += t
        per_step.append(t)
    gbps = moved / dt / 1e9
    line = {"metric": METRIC, "value": gbps, "unit": "GB/s", "impl": "reference", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * dt / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic", "config": workload_config(m, 1, "host"),
            "cpu_baseline": {"value": gbps, "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": f"first 4 of {m.num_layers} layers of each decode step "
                                       f"(memcpy gather, oracle/hv_oracle.c, {threads} threads)"},
            "e2e": {"value": gbps, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line, a)
    return 0


# --------------------------------------------------------------------- GPU path
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


KV_TOKENS, KV_SLAB_BLOCKS = 131072, 64   # BASELINE configs[3]: one 128k-token Llama-3-8B sequence


def kv_slab_bytes():
    from paper_2602_00328_b200.kv import LLAMA3_8B
    return KV_SLAB_BLOCKS * LLAMA3_8B.block_bytes


def kv_long_context(sysm, source, a):
    """Config 4: a 128k-token Llama-3-8B sequence (8,192 blocks x 32 layers x
    64 KiB = 16 GiB) is appended (KV produced locally), evicted out of local
    HBM to harvested peer slabs (N>1, Lossy) or the host tier (N=1, Backed),
    then reloaded with ONE K1 launch of 262,144 pages.  Reports the kernel
    time, the end-to-end reload() time, and a content check of sampled pages."""
    import torch
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.kv import LLAMA3_8B, KVCacheManager, kv_seed
    from paper_2602_00328_b200.runtime import Durability
    m = LLAMA3_8B
    nblk = KV_TOKENS // m.block_tokens
    host = source == "host"
    kv = KVCacheManager(sysm, m, local_blocks=nblk, host_blocks=nblk if host else 1, slab_blocks=KV_SLAB_BLOCKS,
                        durability=Durability.BACKED if host else Durability.LOSSY, engine=a.engine,
                        max_ctas=a.max_ctas)
    kv.append_kv(0, KV_TOKENS)
    t0 = time.perf_counter()
    kv.timing = []
    moves = kv.evict(nblk * m.block_bytes)
    evict_wall = time.perf_counter() - t0
    e_ev0, e_ev1, e_nb = kv.timing[-1]
    where = {}
    for _bid, _frm, to in moves:
        where[to] = where.get(to, 0) + 1
    ids = sorted(kv.table)
    kv.timing = []
    t0 = time.perf_counter()
    plan = kv.reload(ids)
    sysm.engine.synchronize()
    wall = time.perf_counter() - t0
    ev0, ev1, nb = kv.timing[-1]
    ms = ev0.elapsed_time(ev1)
    rng = np.random.default_rng(0)
    sample = [(int(l), int(b)) for l, b in zip(rng.integers(0, m.num_layers, 64), rng.integers(0, nblk, 64))]
    ptrs = [kv.cache[l, kv.table[b].slot].data_ptr() for l, b in sample]
    bad = F.verify_content(F.ptrs_tensor(ptrs, kv.dev), F.ptrs_tensor([m.page_bytes] * len(ptrs), kv.dev),
                           [kv_seed(l, 0, kv.table[b].index) for l, b in sample])
    out = {"sequence_tokens": KV_TOKENS, "blocks": nblk, "pages": nblk * m.num_layers, "bytes": nb,
           "evicted_to": where, "reload_from": {k: len(v) for k, v in plan.items()},
           "reload_kernel_ms": ms, "reload_kernel_GBps": nb / (ms * 1e-3) / 1e9,
           "reload_e2e_ms": wall * 1e3, "evict_kernel_ms": e_ev0.elapsed_time(e_ev1),
           "evict_e2e_ms": evict_wall * 1e3, "sampled_pages_mismatched_words": int(bad.sum()),
           "model": "llama-3-8b: 32 layers x 8 KV heads x 128 x fp16, 16-token blocks"}
    kv.close()
    return out


PROBE_CHILD = r"""
import json, sys
sys.path.insert(0, {repo!r})
import torch
from paper_2602_00328_b200 import fetch as F
from paper_2602_00328_b200.pool import PeerPool
p = PeerPool.import_ipc(bytes.fromhex({handle!r}), {donor}, {nbytes}, {dev})
n = 4 << 20
a = torch.empty(n, dtype=torch.uint8, device="cuda:{dev}")
b = torch.empty(n, dtype=torch.uint8, device="cuda:{dev}")
src = F.ptrs_tensor([p.va], "cuda:{dev}")
sz = F.ptrs_tensor([n], "cuda:{dev}")
F.batch_copy(src, F.ptrs_tensor([a.data_ptr()], "cuda:{dev}"), sz, engine="ldg")
F.batch_copy(src, F.ptrs_tensor([b.data_ptr()], "cuda:{dev}"), sz, engine={engine!r})
torch.cuda.synchronize()
print(json.dumps({{"ok": bool(torch.equal(a, b))}}))
p.close()
"""


def probe_engines_on_peer(handle: bytes, donor: int, nbytes: int, dev: int) -> dict:
    """Run each non-LDG engine on a real peer pointer in a throw-away child
    process: a fault there cannot poison this process's CUDA context."""
    import subprocess
    ok = {"ldg": True}
    for engine in ("ldg256", "tma"):
        code = PROBE_CHILD.format(repo=REPO, handle=handle.hex(), donor=donor, nbytes=nbytes, dev=dev,
                                  engine=engine)
        try:
            r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=180)
            ok[engine] = r.returncode == 0 and '"ok": true' in r.stdout
        except Exception:
            ok[engine] = False
    return ok


def autotune(layer_desc, stream, stream_h, F, reps=3, engines=("ldg", "ldg256", "tma")):
    """Time one layer's real fetch under each engine x grid cap; pick the fastest."""
    import torch
    sp, dp, sz, nb = layer_desc
    rows = []
    for engine in engines:
        for max_ctas in (0, 296, 148):
            for _ in range(1):  # warm
                F.batch_copy(sp, dp, sz, engine=engine, max_ctas=max_ctas, stream=stream_h)
            ts = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                F.batch_copy(sp, dp, sz, engine=engine, max_ctas=max_ctas, stream=stream_h)
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
            rows.append({"engine": engine, "max_ctas": max_ctas, "GBps": nb / statistics.median(ts) / 1e9})
    best = max(rows, key=lambda r: r["GBps"])
    return {"best": best, "candidates": rows}


def run_decode(fetcher, m, dev, world, max_over_ranks, barrier, a, source, microbatches=2, steps=3, warm=2,
               max_ctas=None):
    """MoE decode tokens/s: batch 32 split into `microbatches`, layer-major
    stages, each stage's experts fetched one stage ahead (K2, device-side
    plan) while the previous stage's SwiGLU experts run on the compute stream."""
    import torch
    from paper_2602_00328_b200.decode import MoEDecoder
    dec = MoEDecoder(fetcher, tokens=TOKENS, microbatches=microbatches, seed=7, engine=a.engine,
                     max_ctas=a.max_ctas if max_ctas is None else max_ctas)
    h = dec.decode(warm)
    torch.cuda.synchronize()
    barrier()
    cur = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    h = dec.decode(steps, h)
    e1.record(cur)
    e1.synchronize()
    dt = max_over_ranks(e0.elapsed_time(e1) * 1e-3)
    out = {"tokens_per_s": TOKENS * steps * world / dt, "per_rank_tokens_per_s": TOKENS * steps / dt,
           "batch": TOKENS, "microbatches": microbatches, "steps": steps, "warmup": warm,
           "ms_per_decode_step": dt / steps * 1e3, "expert_source": source,
           "outputs_finite": bool(torch.isfinite(h.float()).all()),
           "model": f"{m.num_layers} MoE layers (router + top-{m.top_k} + SwiGLU experts, bf16); "
                    "attention not modeled"}
    del dec
    return out


def host_offload_decode(m, dev, a, microbatches=1, steps=3, warm=2):
    """The same decode with every expert served from pinned host DRAM (the
    CPU-offload baseline of PAPER.md §4.5), on this GPU."""
    import torch
    from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore
    from paper_2602_00328_b200.pool import HostTier
    from paper_2602_00328_b200.system import HarvestSystem
    host = HostTier(m.num_layers * m.num_experts * m.expert_size)
    sysm = HarvestSystem(dev, host_tier=host, local_bytes=1, engine=a.engine, log_transfers=False)
    store = ExpertStore(m, sysm.host_id, host)
    store.fill_host(dev, weights=True)
    fetcher = ExpertFetcher(sysm.runtime, m, ExpertResidency(m), store)
    r = run_decode(fetcher, m, dev, 1, lambda x: x, lambda: None, a, "host", microbatches, steps, warm)
    sysm.close()
    return r


def same_run_comparisons(dev, m, a, source, fetcher=None, n=53):
    """Same-box comparisons for one layer's worth of experts (n x 17.3 MB):
    the copy-engine paths on the same source (cudaMemcpyBatchAsync: the
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

    out = {}
    dp = F.ptrs_tensor([dst.data_ptr() + i * S for i in range(n)], f"cuda:{dev}")
    sz = F.ptrs_tensor([S] * n, f"cuda:{dev}")
    lp = F.ptrs_tensor([loc.data_ptr() + i * S for i in range(n)], f"cuda:{dev}")
    dt = t(lambda: F.batch_copy(lp, dp, sz, engine=a.engine, stream=s.cuda_stream))
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
                                                sz[:1], engine=a.engine, stream=s.cuda_stream)) * 1e6
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
        lat["kernel_peer"] = t(lambda: F.batch_copy(pdev[:1], dp[:1], sz[:1], engine=a.engine,
                                                    stream=s.cuda_stream)) * 1e6
        lat["copy_engine_peer"] = t(lambda: F.ce_batch_copy(ps[:1], hd[:1], hz[:1], batched=False,
                                                            stream=s.cuda_stream)) * 1e6
        lat["peer_vs_host_speedup"] = lat["copy_engine_host"] / lat["kernel_peer"]
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
    dt_h = t(lambda: F.kv_gather(host_pages, page, dst=kdst, engine=a.engine, stream=s.cuda_stream))
    kv["host_us"], kv["host_GBps"] = dt_h * 1e6, npg * page / dt_h / 1e9
    if source == "peer":
        base = fetcher.src_addr[0, :n]   # peer memory of n experts viewed as page slots
        slots = [int(base[i]) + j * page for i in range(n) for j in range(S // page)]
        peer_pages = F.ptrs_tensor([slots[int(p)] for p in rng.permutation(len(slots))[:npg]], f"cuda:{dev}")
        dt_p = t(lambda: F.kv_gather(peer_pages, page, dst=kdst, engine=a.engine, stream=s.cuda_stream))
        kv["peer_us"], kv["peer_GBps"] = dt_p * 1e6, npg * page / dt_p / 1e9
        kv["peer_vs_host_speedup"] = dt_h / dt_p
    out["kv_config1_layer_gather"] = kv
    out.update(latency_curves(dev, a, s, t, h, fetcher if source == "peer" else None))
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
    from paper_2602_00328_b200.interconnect import calibrate, calibration_rms
    sizes = [65536, 262144, 1 << 20, 4 << 20, 17_301_504]
    dst = torch.empty(max(sizes) + (8000 * 70_272), dtype=torch.uint8, device=f"cuda:{dev}")
    tiers = {"host": host.device_address(0)}
    if fetcher is not None:
        tiers["peer"] = int(fetcher.src_addr[0, 0])
    one = F.ptrs_tensor([S for S in [0]], f"cuda:{dev}")
    curves, fits = {}, {}
    for name, base in tiers.items():
        pts = []
        for nb in sizes:
            sp = F.ptrs_tensor([base], f"cuda:{dev}")
            dp = F.ptrs_tensor([dst.data_ptr()], f"cuda:{dev}")
            sz = F.ptrs_tensor([nb], f"cuda:{dev}")
            pts.append((nb, t(lambda: F.batch_copy(sp, dp, sz, engine=a.engine, stream=s.cuda_stream))))
        curves[name] = [[nb, lat * 1e6] for nb, lat in pts]
        fc, bw = calibrate(pts)
        fits[name] = {"fixed_cost_us": fc * 1e6, "bandwidth_GBps": bw / 1e9, "rms_rel": calibration_rms(pts, fc, bw)}
    out = {"latency_vs_size_us": curves, "calibrated_links": fits}
    if fetcher is not None:
        rows = []
        for model, bpe in (("kimi-k2", 70_272), ("mistral-large-3", 12_800)):   # profiles.py:116-122
            for e in (100, 500, 1000, 2000, 4000, 8000):
                nb = e * bpe
                lat = {}
                for name, base in tiers.items():
                    sp = F.ptrs_tensor([base], f"cuda:{dev}")
                    dp = F.ptrs_tensor([dst.data_ptr()], f"cuda:{dev}")
                    sz = F.ptrs_tensor([nb], f"cuda:{dev}")
                    lat[name] = t(lambda: F.batch_copy(sp, dp, sz, engine=a.engine, stream=s.cuda_stream))
                rows.append([model, e, lat["host"] * 1e6, lat["peer"] * 1e6, lat["host"] / lat["peer"]])
        out["kv_reload_latency_experiment"] = {"columns": ["model", "entries", "host_us", "peer_us", "speedup"],
                                               "rows": rows,
                                               "paper_h100": "kimi-k2 5.42x@100 -> 5.68x@8000 (PAPER.md:319)"}
    del one
    return out


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


def run_b200(a):
    import torch
    import torch.distributed as dist
    from paper_2602_00328_b200 import _native as N
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore, expert_content
    from paper_2602_00328_b200.pool import HostTier, PeerPool
    from paper_2602_00328_b200.runtime import AllocationHints, Durability
    from paper_2602_00328_b200.system import HarvestSystem
    from tools.clocks import ClockSampler

    world = a.gpus
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HV_DEVICE_MAP="0,0" runs several ranks on one GPU (tests of the
    # multi-process IPC path on a single-GPU box; use --dist-backend gloo)
    dmap = os.environ.get("HV_DEVICE_MAP")
    dev = int(dmap.split(",")[local]) if dmap else local
    torch.cuda.set_device(dev)
    backend = a.dist_backend
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
        else:
            dist.init_process_group(backend)
    m = model()
    L, E, S = m.num_layers, m.num_experts, m.expert_size
    routes = routing(m, a.warmup + a.steps, seed=SEED + 1000 * rank)
    imported, host_tier = [], None

    if world == 1:
        source = "host"
        host_tier = HostTier(L * E * S)
        sysm = HarvestSystem(dev, host_tier=host_tier, local_bytes=1, engine=a.engine, max_ctas=a.max_ctas,
                             log_transfers=False)
        store = ExpertStore(m, sysm.host_id, host_tier)
        store.fill_host(dev, weights=True)
        residency = ExpertResidency(m)       # every expert HOST_DRAM
    else:
        source = "peer"
        others = [r for r in range(world) if r != rank]
        per_reader = math.ceil(L * E / (world - 1)) * S
        if not a.no_kv:  # room for config 4's 128k-token KV sequence (128 slabs of 128 MiB)
            per_reader += math.ceil((KV_TOKENS // 16) / KV_SLAB_BLOCKS / (world - 1)) * kv_slab_bytes()
        my_pool = PeerPool(dev, per_reader * (world - 1), readers=[dev], mode="ipc")
        handles = [None] * world
        dist.all_gather_object(handles, my_pool.export_ipc())
        views = {}
        for i, d in enumerate(others, start=1):
            p = PeerPool.import_ipc(handles[d], d, per_reader * (world - 1), dev)
            imported.append(p)
            # my section of donor d: my position among d's readers
            pos = [r for r in range(world) if r != d].index(rank)
            views[i] = p.view(pos * per_reader, per_reader)
        sysm = HarvestSystem(dev, pools=views, local_bytes=1, engine=a.engine, max_ctas=a.max_ctas,
                             log_transfers=False)
        store = ExpertStore(m, sysm.host_id, None)
        residency = ExpertResidency(m)
        rt = sysm.runtime
        # placement: the runtime's own harvest_alloc decisions (runtime.py:198-235);
        # the copy-in is the synthetic-content fill written over NVLink
        ptrs, seeds = [], []
        # round-robin preference (the reference's preferred_devices hint,
        # runtime.py:205-214) so every layer's experts span all N-1 donors and
        # no donor's NVLink egress serves a whole layer alone
        for layer in range(L):
            for e in range(E):
                pref = [1 + (layer * E + e) % (world - 1)]
                h = rt.harvest_alloc(S, AllocationHints(preferred_devices=pref, durability=Durability.BACKED,
                                                        client_id="moe"))
                assert h is not None, "donor capacity exhausted"
                rt.set_tag(h, ("expert", layer, e))
                rt.write_peer(h, ("expert", layer, e), expert_content(m, layer, e))
                residency.set_tier(layer, e, Tier.PEER_HBM, h)
                ptrs.append(rt.address(h))
                seeds.append(expert_content(m, layer, e))
        for i in range(0, len(ptrs), 120):
            F.fill_weights_bf16(F.ptrs_tensor(ptrs[i:i + 120], f"cuda:{dev}"),
                           F.ptrs_tensor([S] * len(ptrs[i:i + 120]), f"cuda:{dev}"), seeds[i:i + 120])
        torch.cuda.synchronize()
        dist.barrier()

    fetcher = ExpertFetcher(sysm.runtime, m, residency, store)
    stream_h = sysm.engine.stream
    stream = torch.cuda.ExternalStream(stream_h, device=f"cuda:{dev}")
    staging = [torch.empty(E * S, dtype=torch.uint8, device=f"cuda:{dev}") for _ in range(2)]
    stage_ptrs = [np.array([b.data_ptr() + i * S for i in range(E)], dtype=np.uint64) for b in staging]

    # ---- device-resident descriptors for the kernel-only (value) loop
    desc = []
    for s in range(a.warmup + a.steps):
        row = []
        for layer in range(L):
            ex = routes[s][layer]
            src = fetcher.src_addr[layer, ex]
            dst = stage_ptrs[layer % 2][:len(ex)]
            row.append((F.ptrs_tensor(src, f"cuda:{dev}"), F.ptrs_tensor(dst, f"cuda:{dev}"),
                        F.ptrs_tensor([S] * len(ex), f"cuda:{dev}"), len(ex) * S))
        desc.append(row)
    torch.cuda.synchronize()

    # ---- engine / grid autotune on the link actually under test (a few launches
    # of one layer's real descriptors); "--engine X" pins the choice instead
    tune = None
    if a.engine == "auto":
        engines = ("ldg", "ldg256", "tma")
        safe = None
        if world > 1:  # engines other than LDG are proven on a peer pointer first, out of process
            if rank == 0:
                d = others[0]
                safe = probe_engines_on_peer(handles[d], d, per_reader * (world - 1), dev)
            box = [safe]
            dist.broadcast_object_list(box, src=0)
            safe = box[0]
            engines = tuple(e for e in engines if safe.get(e))
        tune = autotune(desc[0][0], stream, stream_h, F, engines=engines)
        tune["peer_engine_probe"] = safe
        a.engine, a.max_ctas = tune["best"]["engine"], tune["best"]["max_ctas"]
        if world > 1:  # every rank must run the same configuration: rank 0 decides
            choice = [a.engine, a.max_ctas]
            dist.broadcast_object_list(choice, src=0)
            a.engine, a.max_ctas = choice
        fetcher.engine.engine = N.ENGINES[a.engine]
        fetcher.engine.max_ctas = a.max_ctas

    def value_step(s, evs=None):
        for layer, (sp, dp, sz, nb) in enumerate(desc[s]):
            if evs is not None:
                evs[layer][0].record(stream)
            F.batch_copy(sp, dp, sz, engine=a.engine, max_ctas=a.max_ctas, stream=stream_h)
            if evs is not None:
                evs[layer][1].record(stream)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{dev}" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for s in range(a.warmup):
        value_step(s)
    torch.cuda.synchronize()
    launches0 = N.launch_count()
    step_events = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    for _ in range(L)] for _ in range(a.steps)]
    barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    remeasured = None
    for attempt in range(2):
        with ClockSampler(dev) as clk:
            t0.record(stream)
            for k in range(a.steps):
                value_step(a.warmup + k, step_events[k])
            t1.record(stream)
            t1.synchronize()
        torch.cuda.synchronize()
        bad = clk.summary().get("rejected", False)
        if world > 1:  # every rank re-measures if any rank saw a bad reason
            flag = [bool(bad)]
            flags = [None] * world
            dist.all_gather_object(flags, flag)
            bad = any(f[0] for f in flags)
        if not bad:
            break
        remeasured = clk.summary()  # hw/thermal slowdown seen: keep the record, measure once more
        barrier()
    barrier()
    launches = (N.launch_count() - launches0) // (attempt + 1)   # per timed attempt
    dt = max_over_ranks(t0.elapsed_time(t1) * 1e-3)
    my_bytes = sum(nb for s in range(a.warmup, a.warmup + a.steps) for (_, _, _, nb) in desc[s])
    total_bytes = my_bytes * world
    value = total_bytes / dt / 1e9
    launch_ms = [step_events[k][l][0].elapsed_time(step_events[k][l][1])
                 for k in range(a.steps) for l in range(L)]
    bytes_per_launch = my_bytes / (a.steps * L)
    achieved = bytes_per_launch / (statistics.mean(launch_ms) * 1e-3) / 1e9

    # ---- e2e through the public fetch hook
    seeds_dev = {}

    def e2e_step(s, check):
        fb = None
        for layer in range(L):
            ex = routes[s][layer]
            fb = fetcher.issue_fetches(layer, ex, stage_ptrs[layer % 2][:len(ex)])
        if check:  # verify the last layer against the generator, read counts back
            layer = L - 1
            ex = routes[s][layer]
            key = (s, layer)
            if key not in seeds_dev:
                seeds_dev[key] = F._seeds_tensor([expert_content(m, layer, int(e)) for e in ex], f"cuda:{dev}")
            with torch.cuda.stream(stream):
                bad = F.verify_content(F.ptrs_tensor(stage_ptrs[layer % 2][:len(ex)], f"cuda:{dev}"),
                                       F.ptrs_tensor([S] * len(ex), f"cuda:{dev}"), seeds_dev[key],
                                       stream=stream_h, weights=True)
                host_bad = bad.to("cpu", non_blocking=False)
            return int(host_bad.sum()), len(ex)
        return 0, 0

    for s in range(a.warmup):
        e2e_step(s, True)
    sysm.loop.run()
    barrier()
    torch.cuda.synchronize()
    mism = 0
    d2h = h2d = 0
    w0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(a.steps):
        s = a.warmup + k
        bad, n_last = e2e_step(s, True)
        mism += bad
        d2h += 8 * n_last
        h2d += sum(24 * len(routes[s][layer]) for layer in range(L))
        sysm.loop.poll()
    e1.record(stream)
    e1.synchronize()
    sysm.loop.run()
    wall = time.perf_counter() - w0
    barrier()
    e2e_dt = max_over_ranks(max(wall, e0.elapsed_time(e1) * 1e-3))
    e2e_value = total_bytes / e2e_dt / 1e9
    mism_all = max_over_ranks(float(mism))

    # ---- MoE decode tokens/s through the pipelined decoder (moe.py:211-340)
    del desc
    # one micro-batch: each stage fetches its layer once (fetch-bound path);
    # two micro-batches: the reference's CGOPipe overlap (moe.py:327-340)
    decode = run_decode(fetcher, m, dev, world, max_over_ranks, barrier, a, source, microbatches=1)
    # overlap mode: the fetch kernel's grid is capped so decode compute keeps SMs
    d2 = run_decode(fetcher, m, dev, world, max_over_ranks, barrier, a, source, microbatches=2,
                    max_ctas=a.overlap_max_ctas)
    decode["pipelined_2_microbatches"] = {k: d2[k] for k in ("tokens_per_s", "per_rank_tokens_per_s",
                                                             "ms_per_decode_step", "outputs_finite")}
    decode["pipelined_2_microbatches"]["fetch_max_ctas"] = a.overlap_max_ctas
    sysm.loop.run()
    kvlc = None
    if not a.no_kv:
        kvlc = kv_long_context(sysm, source, a)
        kvlc["reload_kernel_GBps_all_ranks_min"] = -max_over_ranks(-kvlc["reload_kernel_GBps"])
    barrier()
    if world > 1 and rank == 0 and not a.no_host_compare:
        decode["host_offload"] = host_offload_decode(m, dev, a)
        decode["speedup_vs_host_offload_per_gpu"] = (decode["per_rank_tokens_per_s"]
                                                     / decode["host_offload"]["tokens_per_s"])
    barrier()

    if rank == 0:
        if source == "host":
            peak = measure_pcie_h2d(dev)
            roof = {"bound": "pcie", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak if peak else None,
                    "peak_source": "measured in this run: pinned host->device cudaMemcpyAsync, 1 GiB, best of 5"}
        else:
            peak = 770.0
            roof = {"bound": "nvlink", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak,
                    "peak_source": "B200_PROFILING.md fallback: measured peer copy 770 GB/s per direction "
                                   "(900 nominal)"}
        tr = load_traffic().get("batch_copy_" + source)
        roof["traffic"] = tr["traffic_bytes_per_launch"] if tr else None
        if tr:
            roof["traffic_source"] = (f"profiles/traffic.json[{'batch_copy_' + source}]: one ncu --set full capture "
                                      f"({tr['report']}), algorithmic {tr['algorithmic_bytes_per_launch']:.0f} B/launch")
        roof["bytes_per_launch"] = bytes_per_launch
        roof["mean_launch_ms"] = statistics.mean(launch_ms)
        extra = same_run_comparisons(dev, m, a, source, fetcher)
        cpu = None
        if not a.no_cpu_baseline:
            threads = os.cpu_count() or 1
            hc = cpu_host_copy(m, 4 * E)
            gbps, secs, layers, moved = cpu_gather_sample(m, hc, routes[a.warmup:], a.cpu_baseline_s, threads)
            cpu = {"value": gbps, "unit": "GB/s", "cores": threads, "kind": "port",
                   "sample": f"{layers} layer-fetches ({moved / 1e9:.1f} GB) of the same routing, memcpy gather "
                             f"from a host expert table (oracle/hv_oracle.c), {secs:.1f} s, {threads} threads"}
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": 1e3 * dt / a.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
                "config": {**workload_config(m, world, source), "engine": a.engine, "max_ctas": a.max_ctas,
                           "engine_autotune": tune,
                           "parallelism": f"{world} compute GPU(s)" + (f", each reading N-1={world - 1} donors"
                                                                       if world > 1 else "")},
                "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": h2d // a.steps,
                        "d2h_bytes_per_step": d2h // a.steps, "verify_mismatched_words": int(mism_all)},
                "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu,
                "clocks": {**clk.summary(), "first_attempt_rejected": remeasured},
                "latency_ms_per_layer_fetch": statistics.median(launch_ms), "decode": decode,
                "kv_long_context_128k": kvlc, **extra}
    barrier()
    sysm.close()
    for p in imported:
        p.close()
    barrier()
    if world > 1:
        del my_pool  # every reader closed its import above
        import gc
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        phi = None
        if not a.no_phi:
            try:
                phi = phi_phase(world, rank, dev, a, dist, barrier, max_over_ranks)
            except Exception as e:  # report, never lose the main line
                phi = {"error": repr(e)[:300]}
        if rank == 0:
            line["phi35_config3"] = phi
    elif rank == 0:
        line["phi35_config3"] = {"skipped": "config 3 spreads the expert cache over 7 donor B200s; "
                                            "N=1 has no donors (host-tier decode is reported under 'decode')"}
    if not a.no_churn:
        del staging
        torch.cuda.empty_cache()
        try:
            churn = churn_phase(world, rank, dev, a, dist, barrier)
        except Exception as e:
            churn = {"error": repr(e)[:300]}
        if rank == 0:
            line["churn_config5"] = churn
    if rank == 0:
        emit(line, a)
    if world > 1:
        dist.destroy_process_group()
    return 0


def churn_phase(world, rank, dev, a, dist, barrier, layers=8, seconds=2.0):
    """BASELINE configs[4]: donor-memory churn with mid-decode revocation and
    re-placement.  Ranks [0, N/2) are memory-pressured compute GPUs (100% of
    their experts offloaded), ranks [N/2, N) donate HBM.  Every donor follows a
    Markov availability timeline (levels 0/25/50/100% of what it donates, 50 ms
    mean sojourn, seed 5+donor; traces.py:190-213) applied by each compute
    rank's runtime (runtime.py:465-487); revoked experts fall back to the pinned
    host copy and are re-placed by rebalance (moe.py:155-197) when capacity
    returns.  Decode outputs are compared bit-for-bit with an all-local run.
    N=1: the compute GPU donates to itself through a VMM pool."""
    import torch
    from paper_2602_00328_b200.churn import ChurnDriver, expert_tier_counts, markov_availability
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.moe import (QWEN15_MOE_A27B, ExpertFetcher, ExpertResidency, ExpertStore,
                                           MoEProfile, rebalance)
    from paper_2602_00328_b200.pool import HostTier, PeerPool
    from paper_2602_00328_b200.system import HarvestSystem
    from paper_2602_00328_b200.verify import verify_release_ordering
    q = QWEN15_MOE_A27B
    m = MoEProfile(q.name, layers, q.num_experts, q.top_k, q.expert_size, hidden=q.hidden,
                   intermediate=q.intermediate)
    L, E, S = m.num_layers, m.num_experts, m.expert_size
    if world == 1:
        C, D = [0], []
    else:
        C, D = list(range(world // 2)), list(range(world // 2, world))
    n_don = max(1, len(D))
    per_reader = math.ceil(L * E / n_don) * S
    pool, imported, out = None, [], None
    handles = [None] * world
    if world > 1:
        mine = None
        if rank in D:
            try:
                pool = PeerPool(dev, per_reader * len(C), readers=[dev], mode="ipc")
                mine = pool.export_ipc()
            except Exception as e:
                out = {"rank": rank, "error": repr(e)[:200]}
        dist.all_gather_object(handles, mine)
    try:
        if rank in C:
            out = _churn_compute(world, rank, dev, a, m, C, D, per_reader, handles, imported, seconds)
    except Exception as e:  # every rank still reaches the collectives below
        out = {"rank": rank, "error": repr(e)[:300]}
    results = [None] * world
    if world > 1:
        barrier()
        dist.all_gather_object(results, out)
        if pool is not None:
            pool.close()
    else:
        results = [out]
    comp = [r for r in results if r and "error" not in r]
    errs = [r for r in results if r and "error" in r]
    res = {"model": f"{m.name} slice: {L} layers x {E} experts x {S} B (Qwen-shaped, bf16)",
           "compute_ranks": C, "donor_ranks": D if D else "self (VMM pool on the compute GPU)",
           "timeline": "markov_availability levels 0/25/50/100% of the donated bytes, 50 ms mean sojourn, "
                       f"seed 5+donor, {seconds} s",
           "tokens_per_s_all_compute_ranks": sum(r["tokens_per_s"] for r in comp),
           "all_outputs_bit_identical": bool(comp) and all(r["outputs_bit_identical_to_all_local"] for r in comp),
           "total_revocations": sum(r["revocations"] for r in comp),
           "total_re_placements": sum(r["re_placements"] for r in comp),
           "total_release_ordering_violations": sum(r["release_ordering_violations"] for r in comp),
           "per_rank": comp}
    if errs:
        res["errors"] = errs
    return res


def _churn_compute(world, rank, dev, a, m, C, D, per_reader, handles, imported, seconds):
    """Compute-rank side of churn_phase (no collectives inside)."""
    import torch
    from paper_2602_00328_b200.churn import ChurnDriver, expert_tier_counts, markov_availability
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore, rebalance
    from paper_2602_00328_b200.pool import HostTier, PeerPool
    from paper_2602_00328_b200.system import HarvestSystem
    from paper_2602_00328_b200.verify import verify_release_ordering
    L, E, S = m.num_layers, m.num_experts, m.expert_size
    if True:
        host = HostTier(L * E * S)
        if world == 1:
            sysm = HarvestSystem(dev, donors=[dev], donor_bytes=per_reader, host_tier=host, local_bytes=1,
                                 engine=a.engine, max_ctas=a.max_ctas)
        else:
            views = {}
            for i, d in enumerate(D, start=1):
                p = PeerPool.import_ipc(handles[d], d, per_reader * len(C), dev)
                imported.append(p)
                views[i] = p.view(C.index(rank) * per_reader, per_reader)
            sysm = HarvestSystem(dev, pools=views, host_tier=host, local_bytes=1, engine=a.engine,
                                 max_ctas=a.max_ctas)
        rt = sysm.runtime
        store = ExpertStore(m, sysm.host_id, host)
        store.fill_host(dev, weights=True)
        res = ExpertResidency(m)
        counts = np.ones((L, E), dtype=np.int64)
        migrated = [0]

        def replace():
            mig = rebalance(sysm.loop, rt, m, res, counts, sysm.host_id, store=store)
            migrated[0] += len(mig)
            return mig

        replace()
        sysm.loop.run()
        placed0 = expert_tier_counts(res)["PeerHBM"]
        dec = MoEDecoder(ExpertFetcher(rt, m, res, store), tokens=TOKENS, microbatches=1, seed=13,
                         engine=a.engine, max_ctas=a.max_ctas)
        h = dec.step(dec.x0)
        torch.cuda.synchronize()
        GB_levels = [0, per_reader // 4, per_reader // 2, per_reader]
        donors = D if D else [dev]
        drv = ChurnDriver(sysm, {i: markov_availability(GB_levels, [0.05] * 4, seed=5 + d, horizon=seconds)
                                 for i, d in enumerate(donors, start=1)})
        drv.start()
        steps, peer_min, peer_max = 1, placed0, placed0
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            h = dec.step(h)
            steps += 1
            drv.tick(replace)
            pc = expert_tier_counts(res)["PeerHBM"]
            peer_min, peer_max = min(peer_min, pc), max(peer_max, pc)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        sysm.loop.run()
        log = sysm.loop.log
        # all-local reference run of the same number of steps
        resident = torch.from_numpy(host.view()[:L * E * S].copy()).to(f"cuda:{dev}")
        lres = ExpertResidency(m)
        for layer in range(L):
            for e in range(E):
                lres.set_tier(layer, e, Tier.LOCAL_HBM)
        lsys = HarvestSystem(dev, host_bytes=1, local_bytes=1, log_transfers=False)
        lf = ExpertFetcher(lsys.runtime, m, lres, ExpertStore(m, lsys.host_id, None),
                           local_addr=[[resident.data_ptr() + (l * E + e) * S for e in range(E)] for l in range(L)])
        ldec = MoEDecoder(lf, tokens=TOKENS, microbatches=1, seed=13)
        h2 = ldec.x0
        for _ in range(steps):
            h2 = ldec.step(h2)
        torch.cuda.synchronize()
        out = {"rank": rank, "decode_steps": steps - 1, "tokens_per_s": TOKENS * (steps - 1) / wall,
               "availability_steps": len(log.of_kind("availability_step")),
               "revocations": len(log.of_kind("revoke_begin")), "re_placements": migrated[0] - placed0,
               "peer_resident_experts_min_max": [peer_min, peer_max], "experts": L * E,
               "release_ordering_violations": len(verify_release_ordering(log)),
               "outputs_bit_identical_to_all_local": bool(torch.equal(h.view(torch.int16), h2.view(torch.int16)))}
        del dec, ldec, resident
        lsys.close()
        sysm.close()
        for p in imported:
            p.close()
    return out


def phi_phase(world, rank, dev, a, dist, barrier, max_over_ranks, batches=(1, 16, 64)):
    """BASELINE configs[2]: Phi-3.5-MoE-shaped experts (32 layers x 16 experts,
    top-2, 157,286,400 B each) placed by each rank's runtime across its N-1
    donors (up to 7), decode tokens/s at batch 1/16/64.  Rank 0 also times the
    same layers served from pinned host DRAM on a 4-layer slice.
    Collective-safe: local work is guarded, every rank reaches every collective."""
    import torch
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.moe import (PHI35_MOE, ExpertFetcher, ExpertResidency, ExpertStore, MoEProfile,
                                           expert_content)
    from paper_2602_00328_b200.pool import HostTier, PeerPool
    from paper_2602_00328_b200.runtime import AllocationHints, Durability
    from paper_2602_00328_b200.system import HarvestSystem
    m = PHI35_MOE
    if a.phi_layers != m.num_layers:
        m = MoEProfile(m.name, a.phi_layers, m.num_experts, m.top_k, m.expert_size, hidden=m.hidden,
                       intermediate=m.intermediate)
    L, E, S = m.num_layers, m.num_experts, m.expert_size
    others = [r for r in range(world) if r != rank]
    per_reader = math.ceil(L * E / (world - 1)) * S
    out = {"model": f"{m.name}: {L} layers x {E} experts x {S} B, top-{m.top_k}", "donors_per_rank": world - 1}
    errors = []
    pool = sysm = fetcher = None
    imported = []
    try:
        pool = PeerPool(dev, per_reader * (world - 1), readers=[dev], mode="ipc")
        my_handle = pool.export_ipc()
    except Exception as e:
        errors.append(repr(e)[:200])
        my_handle = None
    handles = [None] * world
    dist.all_gather_object(handles, my_handle)
    try:
        if any(h is None for h in handles):
            raise RuntimeError("a donor failed to create its pool")
        views = {}
        for i, d in enumerate(others, start=1):
            p = PeerPool.import_ipc(handles[d], d, per_reader * (world - 1), dev)
            imported.append(p)
            views[i] = p.view([r for r in range(world) if r != d].index(rank) * per_reader, per_reader)
        sysm = HarvestSystem(dev, pools=views, local_bytes=1, engine=a.engine, max_ctas=a.max_ctas,
                             log_transfers=False)
        rt = sysm.runtime
        res = ExpertResidency(m)
        ptrs, seeds = [], []
        for layer in range(L):
            for e in range(E):
                h = rt.harvest_alloc(S, AllocationHints(preferred_devices=[1 + (layer * E + e) % (world - 1)],
                                                        durability=Durability.BACKED, client_id="moe"))
                if h is None:
                    raise RuntimeError("donor capacity exhausted")
                res.set_tier(layer, e, Tier.PEER_HBM, h)
                ptrs.append(rt.address(h))
                seeds.append(expert_content(m, layer, e))
        for i in range(0, len(ptrs), 32):
            F.fill_weights_bf16(F.ptrs_tensor(ptrs[i:i + 32], f"cuda:{dev}"),
                                F.ptrs_tensor([S] * len(ptrs[i:i + 32]), f"cuda:{dev}"), seeds[i:i + 32])
        torch.cuda.synchronize()
        fetcher = ExpertFetcher(rt, m, res, ExpertStore(m, sysm.host_id, None))
    except Exception as e:
        errors.append(repr(e)[:200])
        fetcher = None
    barrier()
    for b in batches:
        dt_local, finite = float("inf"), False
        dec = None
        try:
            if fetcher is None:
                raise RuntimeError("setup failed")
            dec = MoEDecoder(fetcher, tokens=b, microbatches=1, seed=11)
            h = dec.decode(1)
            torch.cuda.synchronize()
        except Exception as e:
            errors.append(repr(e)[:200])
            dec = None
        barrier()
        try:
            if dec is not None:
                cur = torch.cuda.current_stream()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(cur)
                h = dec.decode(3, h)
                e1.record(cur)
                e1.synchronize()
                dt_local = e0.elapsed_time(e1) * 1e-3
                finite = bool(torch.isfinite(h.float()).all())
        except Exception as e:
            errors.append(repr(e)[:200])
        dt = max_over_ranks(dt_local)
        if math.isfinite(dt):
            out[f"batch{b}"] = {"tokens_per_s": b * 3 * world / dt, "per_rank_tokens_per_s": b * 3 / dt,
                                "ms_per_layer": dt / 3 / L * 1e3, "outputs_finite": finite}
        del dec
        torch.cuda.empty_cache()
    if sysm is not None:
        sysm.loop.run()
    if rank == 0 and not a.no_host_compare:
        try:  # host-offload baseline on a 4-layer slice (75 GiB would not fit pinned next to the rest)
            ms = MoEProfile(m.name, 4, E, m.top_k, S, hidden=m.hidden, intermediate=m.intermediate)
            host = HostTier(4 * E * S)
            hsys = HarvestSystem(dev, host_tier=host, local_bytes=1, engine=a.engine, log_transfers=False)
            st = ExpertStore(ms, hsys.host_id, host)
            st.fill_host(dev, weights=True)
            hf = ExpertFetcher(hsys.runtime, ms, ExpertResidency(ms), st)
            for b in batches:
                dec = MoEDecoder(hf, tokens=b, microbatches=1, seed=11)
                dec.decode(1)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                dec.decode(2)
                torch.cuda.synchronize()
                host_ms_layer = (time.perf_counter() - t0) / 2 / 4 * 1e3
                if f"batch{b}" in out:
                    out[f"batch{b}"]["host_offload_ms_per_layer"] = host_ms_layer
                    out[f"batch{b}"]["speedup_vs_host_offload"] = host_ms_layer / out[f"batch{b}"]["ms_per_layer"]
                del dec
            hsys.close()
        except Exception as e:
            out["host_compare_error"] = repr(e)[:300]
    barrier()
    try:
        if sysm is not None:
            sysm.close()
        for p in imported:
            p.close()
    except Exception as e:
        errors.append(repr(e)[:200])
    barrier()
    if pool is not None:
        pool.close()
    all_err = [None] * world
    dist.all_gather_object(all_err, errors)
    if any(all_err):
        out["errors"] = {str(r): e for r, e in enumerate(all_err) if e}
    return out


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    return run_b200(a)


if __name__ == "__main__":
    sys.exit(main())
