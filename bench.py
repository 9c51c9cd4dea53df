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

``value``: descriptor arrays prepared before the timed region; each layer is
one hv_swap_blocks_batch (engine per source: the copy engine for host-tier
experts, the K2 kernel for peer ones) plus its per-fetch content check
(hv_check_digests_batch, read_errors of moe.py:315-319) on a side stream.
``e2e``: the same steps through the public fetch hook
(ExpertFetcher.issue_fetches: host routing -> descriptors staged H2D -> fetch
-> content check), read_errors read back D2H every step.

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

from benchlib.common import (KV_SLAB_BLOCKS, KV_TOKENS, METRIC, SEED, emit, kv_slab_bytes, load_peaks, load_traffic, model, routing, workload_config)  # noqa: E402
from benchlib.compare import (autotune, measure_pcie_h2d, measure_peer_copy, probe_engines_on_peer,  # noqa: E402
                             same_run_comparisons)
from benchlib.cpu import (cpu_gather_sample, cpu_host_copy, cpu_model, reference_simulator, run_reference)  # noqa: E402
from benchlib.phases import (churn_phase, host_offload_decode, kv_decode_config1, kv_long_context,  # noqa: E402
                             offload_sweep_phase, phi_phase, run_decode, all_local_decode)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--engine", default="auto", choices=["auto", "ldg", "ldg256", "ldg16", "tma"])
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--cpu-baseline-s", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--pool-mode", default="remote", choices=["remote", "ipc"],
                    help="N>1 donor pools: VMM chunks donated over Unix sockets, or cudaIpc slabs")
    ap.add_argument("--no-kv", action="store_true", help="skip the config-4 long-context KV measurement")
    ap.add_argument("--no-phi", action="store_true", help="N>1: skip the config-3 Phi-3.5-MoE decode phase")
    ap.add_argument("--no-churn", action="store_true", help="skip the config-5 churn phase")
    ap.add_argument("--no-sweep", action="store_true", help="N=1: skip the host-tier offload-fraction sweep")
    ap.add_argument("--phi-layers", type=int, default=32,
                    help="layers of the Phi-3.5-MoE phase (32 = the real model; fewer only for single-GPU tests)")
    ap.add_argument("--overlap-max-ctas", type=int, default=64,
                    help="fetch grid cap in the 2-micro-batch (overlapped) decode")
    ap.add_argument("--no-host-compare", action="store_true",
                    help="N>1: skip rank 0's host-offload decode comparison")
    a = ap.parse_args()
    a.warmup = max(3, a.warmup)
    return a

def run_b200(a):
    import torch
    import torch.distributed as dist
    from paper_2602_00328_b200 import _native as N
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.cluster import DonorLayout, RankGroup, per_reader_bytes, place_experts
    from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore, expert_content
    from paper_2602_00328_b200.pool import HostTier, NodePools
    from paper_2602_00328_b200.system import HarvestSystem
    from tools.clocks import ClockSampler
    from tools.nvlink_counters import NvlinkCounters
    from tools.nvlink_counters import delta as nvlink_delta

    world = a.gpus
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HV_DEVICE_MAP="0,0" runs several ranks on one GPU (tests of the
    # multi-process IPC path on a single-GPU box; use --dist-backend gloo)
    dmap = os.environ.get("HV_DEVICE_MAP")
    dev = int(dmap.split(",")[local]) if dmap else local

    def device_of(r):   # the CUDA device of rank r (one node: local rank = rank)
        return int(dmap.split(",")[r]) if dmap else r
    torch.cuda.set_device(dev)
    backend = a.dist_backend
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
        else:
            dist.init_process_group(backend)
    group = RankGroup(world, rank, device=f"cuda:{dev}" if backend == "nccl" else None)
    a.group, a.device_of = group, device_of     # for the multi-rank phases
    m = model()
    L, E, S = m.num_layers, m.num_experts, m.expert_size
    routes = routing(m, a.warmup + a.steps, seed=SEED + 1000 * rank)
    host_tier, node = None, None

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
        per_reader = per_reader_bytes(L * E, S, world - 1)
        if not a.no_kv:  # room for config 4's 128k-token KV sequence (128 slabs of 128 MiB)
            per_reader += math.ceil((KV_TOKENS // 16) / KV_SLAB_BLOCKS / (world - 1)) * kv_slab_bytes()
        layout = DonorLayout.symmetric(world, per_reader)
        others = layout.donors_of(rank)
        # donor pools: VMM chunks donated per reader over Unix sockets (HBM
        # goes back to the donor on free / revoke), or cudaIpc slabs
        node = NodePools(group, layout, rank, device_of, mode=a.pool_mode, tag="main")
        views = node.views
        sysm = HarvestSystem(dev, pools=views, local_bytes=1, engine=a.engine, max_ctas=a.max_ctas,
                             log_transfers=False)
        store = ExpertStore(m, sysm.host_id, None)
        residency = ExpertResidency(m)
        rt = sysm.runtime
        # placement: the runtime's own harvest_alloc decisions (runtime.py:198-235)
        # with a rank-offset round-robin donor preference (cluster.preferred_peer);
        # the copy-in is the synthetic-content fill written over NVLink
        placed, seeds = place_experts(rt, m, residency, rank, world - 1)
        ptrs = [rt.address(h) for h in placed]
        for i in range(0, len(ptrs), 120):
            F.fill_weights_bf16(F.ptrs_tensor(ptrs[i:i + 120], f"cuda:{dev}"),
                           F.ptrs_tensor([S] * len(ptrs[i:i + 120]), f"cuda:{dev}"), seeds[i:i + 120])
        torch.cuda.synchronize()
        group.barrier()

    fetcher = ExpertFetcher(sysm.runtime, m, residency, store)
    stream_h = sysm.engine.stream
    stream = torch.cuda.ExternalStream(stream_h, device=f"cuda:{dev}")
    staging = [torch.empty(E * S, dtype=torch.uint8, device=f"cuda:{dev}") for _ in range(2)]
    stage_ptrs = [np.array([b.data_ptr() + i * S for i in range(E)], dtype=np.uint64) for b in staging]

    # ---- per-fetch content identity (read_errors, moe.py:315-319): digests of
    # the authoritative copies -- the pinned host tier at N=1, the placed donor
    # copies at N>1 (written by the fill above, never modified)
    if host_tier is not None:
        expected = store.host_digests(dev)
    else:
        expected = np.empty((L, E), dtype=np.uint64)
        szs = F.ptrs_tensor([S] * E, f"cuda:{dev}")
        for layer in range(L):
            expected[layer] = F.digest(F.ptrs_tensor(fetcher.src_addr[layer], f"cuda:{dev}"), szs).cpu().numpy().view(np.uint64)
    check_s = torch.cuda.Stream(device=f"cuda:{dev}")
    fetcher.enable_content_check(expected, stream=check_s)

    # ---- host descriptor arrays for the fetch-only (value) loop: what the
    # fetch hook would hand the library, prepared before the timed region
    desc = []
    for s in range(a.warmup + a.steps):
        row = []
        for layer in range(L):
            ex = routes[s][layer]
            row.append((np.ascontiguousarray(fetcher.src_addr[layer, ex]),
                        np.ascontiguousarray(stage_ptrs[layer % 2][:len(ex)]),
                        np.full(len(ex), S, dtype=np.uint64), len(ex) * S,
                        np.ascontiguousarray(expected[layer, ex])))
        desc.append(row)
    torch.cuda.synchronize()

    # ---- engine / grid autotune on the link actually under test (a few launches
    # of one layer's real descriptors); "--engine X" pins the choice instead
    tune = None

    barrier = group.barrier
    max_over_ranks = group.max
    chk_scratch = torch.zeros(E, dtype=torch.int64, device=f"cuda:{dev}")
    chk_errors = torch.zeros(1, dtype=torch.int64, device=f"cuda:{dev}")
    a.kernel_engine = a.engine if a.engine not in ("ce", "auto") else "auto"

    if a.engine == "auto":
        engines = ("ldg", "ldg256", "ldg16", "tma")
        safe = None
        if world > 1:  # engines other than LDG are proven on a peer pointer first, out of process
            if rank == 0:
                d = others[0]
                safe = probe_engines_on_peer(node, d, device_of(d), dev)
            safe = group.decide(safe)
            engines = tuple(e for e in engines if safe.get(e))
            # N-1 donors: also the interleaved chunk order (HV_ENGINE_FLAG_INTERLEAVE),
            # which keeps every donor's egress busy instead of all readers
            # walking the same donors in the same order
            engines = engines + tuple(e + "+il" for e in engines)
        # plus the copy engine and the library's engine per source
        tune = autotune(desc[0][0], stream, stream_h, F, engines=engines + ("ce", "auto"),
                        barrier=barrier if world > 1 else None,
                        max_over_ranks=max_over_ranks if world > 1 else None,
                        checked=(chk_scratch, chk_errors) if source == "peer" else None)
        tune["peer_engine_probe"] = safe
        kern = [r for r in tune["candidates"] if r["engine"] not in ("ce", "auto")]
        kbest = max(kern, key=lambda r: r["GBps"])
        a.engine, a.max_ctas = tune["best"]["engine"], tune["best"]["max_ctas"]
        a.kernel_engine = kbest["engine"]
        # every rank must run the same configuration: rank 0 decides
        a.engine, a.max_ctas, a.kernel_engine = group.decide([a.engine, a.max_ctas, a.kernel_engine])
        fetcher.engine.engine = N.ENGINES[a.engine]
        fetcher.engine.max_ctas = a.max_ctas

    fetch_done = [torch.cuda.Event() for _ in range(L)]
    check_done = [torch.cuda.Event() for _ in range(L)]
    eng_code = N.ENGINES[a.engine]
    # the product's choice (ExpertFetcher.issue_fetches): a stage with peer
    # experts is fetched and checked in one kernel pass; an all-host stage
    # rides the copy engine with the digest on a side stream
    fused_check = source == "peer"

    def value_step(s, evs=None):
        """One decode step's fetches: per layer, one hv_swap_blocks_batch on the
        fetch stream, then its content check on the check stream (beside the
        next layer's fetch); staging buffer layer%2 is refilled only after the
        check of two layers back has read it."""
        for layer, (sp, dp, sz, nb, ex_d) in enumerate(desc[s]):
            if fused_check:   # peer tier: fetch + digest in one kernel pass, compare on the same stream
                if evs is not None:
                    evs[layer][0].record(stream)
                N.call("hv_swap_blocks_batch_checked", sp.ctypes.data, dp.ctypes.data, sz.ctypes.data,
                       ex_d.ctypes.data, len(sp), eng_code, a.max_ctas, chk_scratch.data_ptr(), 0,
                       chk_errors.data_ptr(), stream_h)
                if evs is not None:
                    evs[layer][1].record(stream)
                continue
            if layer >= 2:
                stream.wait_event(check_done[layer - 2])
            if evs is not None:
                evs[layer][0].record(stream)
            N.call("hv_swap_blocks_batch", sp.ctypes.data, dp.ctypes.data, sz.ctypes.data, len(sp), eng_code,
                   a.max_ctas, stream_h)
            if evs is not None:
                evs[layer][1].record(stream)
            fetch_done[layer].record(stream)
            check_s.wait_event(fetch_done[layer])
            if evs is not None:
                evs[layer][2].record(check_s)
            N.call("hv_check_digests_batch", dp.ctypes.data, sz.ctypes.data, ex_d.ctypes.data, len(sp),
                   chk_scratch.data_ptr(), 0, chk_errors.data_ptr(), check_s.cuda_stream)
            if evs is not None:
                evs[layer][3].record(check_s)
            check_done[layer].record(check_s)
        if not fused_check:
            stream.wait_event(check_done[L - 1])
            stream.wait_event(check_done[L - 2])

    for s in range(a.warmup):
        value_step(s)
    torch.cuda.synchronize()
    launches0 = N.launch_count()
    step_events = [[tuple(torch.cuda.Event(enable_timing=True) for _ in range(4))
                    for _ in range(L)] for _ in range(a.steps)]
    barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    remeasured = None
    nvl = NvlinkCounters(dev)
    for attempt in range(2):
        with ClockSampler(dev) as clk:
            nv0 = nvl.snapshot()
            t0.record(stream)
            for k in range(a.steps):
                value_step(a.warmup + k, step_events[k])
            t1.record(stream)
            t1.synchronize()
            nv1 = nvl.snapshot()
        torch.cuda.synchronize()
        # hardware NVLink byte counters of this GPU over the timed region
        nvlink = nvlink_delta(nv0, nv1, t0.elapsed_time(t1) * 1e-3)
        bad = clk.summary().get("rejected", False)
        bad = group.any(bad)  # every rank re-measures if any rank saw a bad reason
        if not bad:
            break
        remeasured = clk.summary()  # hw/thermal slowdown seen: keep the record, measure once more
        barrier()
    barrier()
    launches = (N.launch_count() - launches0) // (attempt + 1)   # per timed attempt
    value_read_errors = int(chk_errors.item())
    my_dt = t0.elapsed_time(t1) * 1e-3
    dt = max_over_ranks(my_dt)
    my_bytes = sum(d[3] for s in range(a.warmup, a.warmup + a.steps) for d in desc[s])
    per_rank = group.all_gather((my_bytes, my_dt))     # each rank's own routing -> its own byte count
    total_bytes = sum(nb for nb, _ in per_rank)
    value = total_bytes / dt / 1e9
    launch_ms = [step_events[k][l][0].elapsed_time(step_events[k][l][1])
                 for k in range(a.steps) for l in range(L)]
    check_ms = None if fused_check else [step_events[k][l][2].elapsed_time(step_events[k][l][3])
                                         for k in range(a.steps) for l in range(L)]
    bytes_per_launch = my_bytes / (a.steps * L)
    achieved = bytes_per_launch / (statistics.mean(launch_ms) * 1e-3) / 1e9

    # ---- e2e through the public fetch hook (ExpertFetcher.issue_fetches with
    # its per-fetch content check), read_errors read back D2H every step
    def e2e_step(s):
        batches = []
        for layer in range(L):
            ex = routes[s][layer]
            if layer >= 2:
                batches[layer - 2].wait_on(stream)   # staging buffer reuse: after that stage's check
            batches.append(fetcher.issue_fetches(layer, ex, stage_ptrs[layer % 2][:len(ex)]))
        return fetcher.read_errors()

    for s in range(a.warmup):
        e2e_step(s)
    sysm.loop.run()
    errors0 = fetcher.read_errors()
    barrier()
    torch.cuda.synchronize()
    d2h = h2d = 0
    w0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(a.steps):
        s = a.warmup + k
        errors = e2e_step(s)
        d2h += 8                                   # the read_errors counter
        nobj = sum(len(routes[s][layer]) for layer in range(L))
        h2d += 16 * nobj + 24 * nobj               # fetch (src, dst) + check (dst, size, digest) descriptors
        if source == "host":                       # the step's inputs: expert bytes read from pinned host memory
            h2d += nobj * S
        sysm.loop.poll()
    e1.record(stream)
    e1.synchronize()
    sysm.loop.run()
    wall = time.perf_counter() - w0
    barrier()
    e2e_dt = max_over_ranks(max(wall, e0.elapsed_time(e1) * 1e-3))
    e2e_value = total_bytes / e2e_dt / 1e9
    read_errors_all = max_over_ranks(float(errors - errors0 + value_read_errors))
    # untimed: the last stage's bytes against the content generator itself
    # (the read_errors digests are relative to the authoritative copy)
    ex = routes[a.warmup + a.steps - 1][L - 1]
    vbad = F.verify_content(F.ptrs_tensor(stage_ptrs[(L - 1) % 2][:len(ex)], f"cuda:{dev}"),
                            F.ptrs_tensor([S] * len(ex), f"cuda:{dev}"),
                            [expert_content(m, L - 1, int(e)) for e in ex], weights=True)
    mism_all = max_over_ranks(float(vbad.sum().item()))
    nvlink_all = group.all_gather(nvlink)

    # ---- MoE decode tokens/s through the pipelined decoder (moe.py:211-340)
    del desc
    # one micro-batch: each stage fetches its layer once (fetch-bound path);
    # two micro-batches: the reference's CGOPipe overlap (moe.py:327-340)
    decode = run_decode(fetcher, m, dev, world, max_over_ranks, barrier, a, source, microbatches=1)
    # overlap mode: the fetch kernel's grid is capped so decode compute keeps SMs
    d2 = run_decode(fetcher, m, dev, world, max_over_ranks, barrier, a, source, microbatches=2,
                    max_ctas=a.overlap_max_ctas)
    decode["pipelined_2_microbatches"] = {k: d2.get(k) for k in ("tokens_per_s", "per_rank_tokens_per_s",
                                                                 "ms_per_decode_step", "outputs_finite",
                                                                 "overlap")}
    decode["pipelined_2_microbatches"]["fetch_max_ctas"] = a.overlap_max_ctas
    # the same decode consuming every expert in place (fused fetch + FFN)
    try:
        decode["fused"] = run_decode(fetcher, m, dev, world, max_over_ranks, barrier, a, source, microbatches=1,
                                     fused=True)
    except Exception as e:  # report, never lose the line (every rank reaches the same collectives)
        decode["fused"] = {"error": repr(e)[:300]}
    if source == "host":   # N=1: the host-tier fetch through the copy engine (plan read back per stage)
        try:
            decode["host_plan"] = run_decode(fetcher, m, dev, world, max_over_ranks, barrier, a, source,
                                             microbatches=1, host_plan=True)
        except Exception as e:
            decode["host_plan"] = {"error": repr(e)[:300]}
        try:   # the same decoder with every expert in HBM: its compute ceiling (not an offload mode)
            decode["all_local_ceiling"] = all_local_decode(sysm, store, m, dev)
        except Exception as e:
            decode["all_local_ceiling"] = {"error": repr(e)[:300]}
    # the faster of the measured decode modes (each one bit-identical to its all-local run)
    modes = {"staged": decode.get("tokens_per_s"), "staged_cuda_graph": (decode.get("cuda_graph") or {}).get("tokens_per_s"),
             "fused": decode["fused"].get("tokens_per_s"),
             "fused_cuda_graph": (decode["fused"].get("cuda_graph") or {}).get("tokens_per_s"),
             "staged_host_plan": (decode.get("host_plan") or {}).get("tokens_per_s")}
    modes = {k: v for k, v in modes.items() if v}
    if modes:
        best = max(modes, key=modes.get)
        decode["best"] = {"mode": best, "tokens_per_s": modes[best]}
    sysm.loop.run()
    kvlc = None
    kvd1 = None
    if not a.no_kv:
        try:
            kvd1 = kv_decode_config1(sysm, source, a)
        except Exception as e:  # report, never lose the line
            kvd1 = {"error": repr(e)[:300]}
        try:
            kvlc = kv_long_context(sysm, source, a)
        except Exception as e:   # reported; every rank still reaches the collective below
            kvlc = {"error": repr(e)[:300]}
        kvlc["reload_kernel_GBps_all_ranks_min"] = -max_over_ranks(-kvlc.get("reload_kernel_GBps", 0.0))
    barrier()
    if world > 1 and rank == 0 and not a.no_host_compare:
        try:   # rank 0 alone, between barriers: a failure is reported, never a hang
            decode["host_offload"] = host_offload_decode(m, dev, a)
            decode["speedup_vs_host_offload_per_gpu"] = (decode["per_rank_tokens_per_s"]
                                                         / decode["host_offload"]["tokens_per_s"])
            if "best" in decode:
                decode["best"]["speedup_vs_host_offload_per_gpu"] = (decode["best"]["tokens_per_s"] / world
                                                                     / decode["host_offload"]["tokens_per_s"])
        except Exception as e:
            decode["host_offload"] = {"error": repr(e)[:300]}
    barrier()

    if rank == 0:
        if source == "host":
            peak = measure_pcie_h2d(dev)
            roof = {"bound": "pcie", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak if peak else None,
                    "peak_source": "measured in this run: pinned host->device cudaMemcpyAsync, 1 GiB, best of 5"}
        else:
            donor_dev = device_of(layout.donors_of(rank)[0])
            meas = measure_peer_copy(dev, donor_dev)
            peak = meas or 770.0
            roof = {"bound": "nvlink", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak,
                    "peak_source": (f"measured in this run: cudaMemcpyPeerAsync GPU {donor_dev} -> GPU {dev}, "
                                    "256 MiB, best of 5" if meas else
                                    "B200_PROFILING.md fallback: measured peer copy 770 GB/s per direction "
                                    "(900 nominal); the donor is this GPU (single-GPU stand-in)")}
        roof["engine"] = a.engine
        if a.engine in ("ce", "auto") and source == "host":
            # the copy engine moves the host-tier experts: a DMA engine, not a
            # kernel -- ncu has nothing to capture; the step's SM kernel is the
            # per-fetch check, reported in roofline_check_kernel
            roof["traffic"] = None
            roof["traffic_source"] = ("copy engine (cudaMemcpyAsync): not a kernel, no ncu capture; the same "
                                      "bytes through the K2 kernel: profiles/traffic.json[batch_copy_host]")
        elif source == "peer":
            # one GPU per gpurun call: no capture of a peer source exists; the
            # same kernel on an HBM source is the nearest evidence
            trh = load_traffic().get("checked_hbm_" + str(a.engine).split("+")[0])
            roof["traffic"] = None
            roof["traffic_source"] = ("no ncu capture of a peer (NVLink) source on a 1-GPU box; the same fused "
                                      "fetch+check kernel on an HBM source: " +
                                      (f"profiles/traffic.json[checked_hbm_{str(a.engine).split('+')[0]}] "
                                       f"= {trh['traffic_bytes_per_launch']:.0f} B per "
                                       f"{trh['algorithmic_bytes_per_launch']:.0f} algorithmic" if trh else
                                       "not captured for this engine"))
        else:
            tr = load_traffic().get("batch_copy_" + source)
            roof["traffic"] = tr["traffic_bytes_per_launch"] if tr else None
            if tr:
                roof["traffic_source"] = (f"profiles/traffic.json[{'batch_copy_' + source}]: one ncu --set full "
                                          f"capture ({tr['report']}), algorithmic "
                                          f"{tr['algorithmic_bytes_per_launch']:.0f} B/launch")
        roof["bytes_per_launch"] = bytes_per_launch
        roof["mean_launch_ms"] = statistics.mean(launch_ms)
        hbm_peak = load_peaks().get("hbm_gbs")
        trc = load_traffic().get("check_digests")
        if check_ms is None:
            roof_check = {"kernel": "fused into the fetch kernel (hv_swap_blocks_batch_checked: CopyDigestOp digests "
                                    "every 16 B it moves); see roofline", "separate_launch": False}
            trc = None
        else:
            chk_gbps = bytes_per_launch / (statistics.mean(check_ms) * 1e-3) / 1e9
            roof_check = {"kernel": "hv_check_digests (digest of every arrival + compare; desc_digest_tma + "
                                    "digest_compare_kernel), beside the copy engine on a side stream",
                          "bound": "hbm", "achieved": chk_gbps,
                          "peak": hbm_peak, "unit": "GB/s", "frac": chk_gbps / hbm_peak if hbm_peak else None,
                          "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, read+write; this kernel only reads)",
                          "bytes_per_launch": bytes_per_launch, "mean_launch_ms": statistics.mean(check_ms),
                          "traffic": trc["traffic_bytes_per_launch"] if trc else None}
        if trc:
            roof_check["traffic_source"] = f"profiles/traffic.json[check_digests] ({trc['report']})"
        try:   # rank-0 local work only (no collectives inside): a failure is reported, never fatal
            extra = same_run_comparisons(dev, m, a, source, fetcher)
        except Exception as e:
            extra = {"same_run_comparisons_error": repr(e)[:300]}
        # the copy engine on the same source, measured in this run, beside the peak
        # the fraction is taken against (a second, in-run ceiling for the reader)
        ce = extra.get("copy_engine_same_source_GBps")
        if ce:
            roof["copy_engine_same_source_GBps"] = ce
            roof["frac_of_copy_engine_same_source"] = achieved / ce
        cpu = None
        if world > 1:   # the CPU restatement is timed on rank 0 at N=1 only (contract)
            cpu = {"skipped": "timed in the N=1 run (rank 0, host cores)"}
        elif not a.no_cpu_baseline:
            threads = os.cpu_count() or 1
            hc = cpu_host_copy(m, 4 * E)
            gbps, secs, layers, moved = cpu_gather_sample(m, hc, routes[a.warmup:], a.cpu_baseline_s, threads)
            cpu = {"value": gbps, "unit": "GB/s", "cores": threads, "kind": "port",
                   "sample": f"{layers} layer-fetches ({moved / 1e9:.1f} GB) of the same routing, memcpy gather "
                             f"from a host expert table (oracle/hv_oracle.c), {secs:.1f} s, {threads} threads"}
            g1, s1, l1, _ = cpu_gather_sample(m, hc, routes[a.warmup:], min(5.0, a.cpu_baseline_s), 1)
            cpu["single_thread"] = {"value": g1, "unit": "GB/s", "cores": 1, "sample": f"{l1} layer-fetches, {s1:.1f} s"}
            cpu["cpu_model"] = cpu_model()
        try:
            refsim = reference_simulator(m, world - 1)
        except Exception as e:  # report, never lose the main line
            refsim = {"error": repr(e)[:300]}
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": 1e3 * dt / a.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
                "config": workload_config(m, world),
                "implementation": {"source_tier": source, "donors_per_rank": max(0, world - 1),
                                   "engine": a.engine, "max_ctas": a.max_ctas, "kernel_engine": a.kernel_engine,
                                   "engine_autotune": tune,
                                   "parallelism": f"{world} compute GPU(s)" + (
                                       f", each reading N-1={world - 1} donors" if world > 1 else "")},
                "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": h2d // a.steps,
                        "d2h_bytes_per_step": d2h // a.steps, "read_errors": int(read_errors_all),
                        "verify_mismatched_words": int(mism_all),
                        "read_errors_note": "objects whose fetched bytes' digest differed from the authoritative "
                                            "copy's, over every fetch of the timed value and e2e steps "
                                            "(moe.py:315-319)"},
                "gpu_launches": launches, "roofline": roof, "roofline_check_kernel": roof_check,
                "cpu_baseline": cpu,
                "clocks": {**clk.summary(), "first_attempt_rejected": remeasured},
                "latency_ms_per_layer_fetch": statistics.median(launch_ms),
                "latency_ms_per_layer_fetch_dist": {"p50": float(np.percentile(launch_ms, 50)),
                                                    "p99": float(np.percentile(launch_ms, 99)),
                                                    "n": len(launch_ms)}, "decode": decode,
                "kv_long_context_128k": kvlc, "kv_decode_config1": kvd1, "reference_simulator": refsim,
                "per_rank_GBps": [nb / t / 1e9 for nb, t in per_rank],
                "nvlink_counters_timed_region": {
                    "per_rank": nvlink_all,
                    "note": "NVML per-link NVLink data counters of each rank's GPU, read before/after the timed "
                            "fetch steps (rx = bytes this GPU pulled from donors, tx = bytes it served)"},
                **extra}
    barrier()
    sysm.close()
    if node is not None:
        pool_info = {"mode": node.mode, "setup_error": node.error, "fallback_reason": node.fallback_reason}
        node.close()
        if rank == 0:
            line["implementation"]["donor_pools"] = pool_info
    barrier()
    if world > 1:
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
            churn = churn_phase(world, rank, dev, a, dist, barrier,
                                seconds=float(os.environ.get("HV_CHURN_SECONDS", "2.0")))
        except Exception as e:
            churn = {"error": repr(e)[:300]}
        if rank == 0:
            line["churn_config5"] = churn
    if rank == 0 and world == 1 and not a.no_sweep:
        try:   # rank 0, N=1 only: local work, no collectives
            line["offload_sweep"] = offload_sweep_phase(m, dev, a)
        except Exception as e:
            line["offload_sweep"] = {"error": repr(e)[:300]}
    if rank == 0:
        line["north_star_targets"] = north_star_targets(line, world)
        emit(line, a)
    if world > 1:
        dist.destroy_process_group()
    return 0

def north_star_targets(line, world):
    """BASELINE.json north_star targets read off this line (measured values
    only; a target whose inputs this N does not produce says so)."""
    out = {}
    roof = line.get("roofline") or {}
    if world > 1:
        out["peer_fetch_frac_of_nvlink"] = {"value": roof.get("frac"), "target": ">= 0.80",
                                            "source": "roofline.achieved / roofline.peak (" +
                                                      str(roof.get("peak_source", "")) + ")"}
    else:
        out["peer_fetch_frac_of_nvlink"] = {"value": None, "note": "N=1 has no donor: host tier only"}
    lat = line.get("single_expert_latency_us") or {}
    out["fetch_latency_host_over_peer"] = {"value": lat.get("peer_vs_host_speedup"), "target": ">= 5",
                                           "source": "single 17.3 MB expert, K2 kernel, host vs peer"}
    kv = line.get("kv_config1_layer_gather") or {}
    out["kv_page_fetch_host_over_peer"] = {"value": kv.get("peer_vs_host_speedup"), "target": ">= 5",
                                           "source": "config-1 layer gather, 1,024 x 64 KiB pages"}
    dec = (line.get("decode") or {}).get("best") or {}
    out["moe_decode_vs_host_offload"] = {"value": dec.get("speedup_vs_host_offload_per_gpu"), "target": ">= 1.5",
                                         "mode": dec.get("mode"),
                                         "source": "per-GPU decode tok/s, peer tiers vs the same GPU's host offload"}
    if os.environ.get("HV_DEVICE_MAP"):
        out["stand_in"] = ("HV_DEVICE_MAP: several ranks share one GPU and the 'peers' are IPC imports of "
                           "that GPU's own HBM, so link fractions and ratios here are HBM, not NVLink, figures")
    out["bit_exact"] = {"fetch_read_errors": (line.get("e2e") or {}).get("read_errors"),
                        "decode_outputs_equal_all_local_under_churn":
                            (line.get("churn_config5") or {}).get("all_outputs_bit_identical")}
    return out


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    try:
        return run_b200(a)
    except Exception as e:   # say what failed on stdout (rank 0), then fail the run
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps({"metric": METRIC, "value": None, "n_gpus": a.gpus, "error": repr(e)[:500]}),
                  flush=True)
        raise


if __name__ == "__main__":
    sys.exit(main())
