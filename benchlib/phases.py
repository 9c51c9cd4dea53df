"""Benchmark phases beyond the headline fetch: MoE decode (configs[1]/[2]), long-context KV
(configs[3]) and donor churn (configs[4])."""
from __future__ import annotations

import math
import time

import numpy as np

from benchlib.common import KV_SLAB_BLOCKS, KV_TOKENS, TOKENS


def run_decode(fetcher, m, dev, world, max_over_ranks, barrier, a, source, microbatches=2, steps=3, warm=2,
               max_ctas=None, fused=False, host_plan=False):
    """MoE decode tokens/s: batch 32 split into `microbatches`, layer-major
    stages, each stage's experts fetched one stage ahead (K2, device-side
    plan) while the previous stage's SwiGLU experts run on the compute stream."""
    import torch
    from paper_2602_00328_b200.decode import MoEDecoder
    dec = MoEDecoder(fetcher, tokens=TOKENS, microbatches=microbatches, seed=7, engine=getattr(a, "kernel_engine", a.engine),
                     max_ctas=a.max_ctas if max_ctas is None else max_ctas, fused=fused, host_plan=host_plan)
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
    if fused:
        out["mode"] = ("fused: experts consumed in place (hv_expert_ffn_gate_up/down stream weight tiles from "
                       "the resident copy into tcgen05.mma; host-tier experts staged by K2 first)")
    if host_plan:
        out["mode"] = ("staged, host plan: each stage's plan read back once routed and fetched through the engine per "
                       "source (copy engine for host-tier experts); eager only")
        del dec
        return out
    if microbatches > 1 and not fused:  # one extra, traced step: device-clock proof of fetch/compute overlap
        dec.trace = True
        dec.step(h)
        out["overlap"] = dec.overlap_report()
    else:  # the same step as one CUDA graph replay (no per-launch host cost)
        try:
            h_eager = dec.step(h).clone()
            dec.capture_graph()
            same = bool(torch.equal(dec.step(h).view(torch.int16), h_eager.view(torch.int16)))
            torch.cuda.synchronize()
            barrier()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(cur)
            hg = h_eager
            for _ in range(steps):
                hg = dec.step(hg)
            g1.record(cur)
            g1.synchronize()
            dtg = max_over_ranks(g0.elapsed_time(g1) * 1e-3)
            out["cuda_graph"] = {"tokens_per_s": TOKENS * steps * world / dtg,
                                 "ms_per_decode_step": dtg / steps * 1e3,
                                 "replay_equals_eager_bitwise": same}
        except Exception as e:  # report, never lose the line
            out["cuda_graph"] = {"error": repr(e)[:300]}
    del dec
    return out

def all_local_decode(sysm, store, m, dev, steps=5, warm=2):
    """The decoder's compute ceiling: every expert resident in this GPU's HBM
    (the host tier's bytes copied once), fused decode as one CUDA graph per
    step, experts row-major and then stored as HV_FFN_TILED tiles (the same
    logical weights: outputs must be bit-identical).  Not an offload number --
    it bounds what any tier can deliver to this decoder."""
    import torch
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore
    L, E, S, H, I = m.num_layers, m.num_experts, m.expert_size, m.hidden, m.intermediate
    view = store.host.view()
    resident = torch.empty(L * E * S, dtype=torch.uint8, device=f"cuda:{dev}")
    step = E * S
    for o in range(0, L * E * S, step):
        resident[o:o + step].copy_(torch.from_numpy(view[store.base_offset + o:store.base_offset + o + step]))
    res = ExpertResidency(m)
    for layer in range(L):
        for e in range(E):
            res.set_tier(layer, e, Tier.LOCAL_HBM)
    addr = [[resident.data_ptr() + (layer * E + e) * S for e in range(E)] for layer in range(L)]
    out, ref = {"model": f"{m.name}: {L} layers x {E} experts, batch {TOKENS}, top-{m.top_k}",
                "expert_source": "local HBM (all resident)", "mode": "fused, CUDA graph per step"}, None
    for layout in ("row", "tiled"):
        if layout == "tiled":
            for o in range(0, L * E * S, S):
                w = resident[o:o + S].view(torch.bfloat16)
                t = torch.cat([F.tile_expert_matrix(w[:I * H].view(I, H)).reshape(-1),
                               F.tile_expert_matrix(w[I * H:2 * I * H].view(I, H)).reshape(-1),
                               F.tile_expert_matrix(w[2 * I * H:].view(H, I)).reshape(-1)])
                w.copy_(t)
        lstore = ExpertStore(m, store.host_device_id, None)
        lstore.layout = layout
        f = ExpertFetcher(sysm.runtime, m, res, lstore, local_addr=addr)
        dec = MoEDecoder(f, tokens=TOKENS, microbatches=1, seed=7, fused=True)
        h = dec.decode(warm)
        dec.capture_graph()
        h0 = h.clone()
        for _ in range(warm):
            h = dec.step(h)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur)
        hg = h
        for _ in range(steps):
            hg = dec.step(hg)
        e1.record(cur)
        e1.synchronize()
        dt = e0.elapsed_time(e1) * 1e-3
        one = dec.step(h0).clone()
        torch.cuda.synchronize()
        if ref is None:
            ref = one
        out[layout] = {"tokens_per_s": TOKENS * steps / dt, "ms_per_decode_step": dt / steps * 1e3,
                       "equals_row_major_bitwise": bool(torch.equal(one.view(torch.int16), ref.view(torch.int16)))}
        del dec, f
    del resident
    torch.cuda.empty_cache()
    return out


def host_offload_decode(m, dev, a, microbatches=1, steps=3, warm=2):
    """The same decode with every expert served from pinned host DRAM (the
    CPU-offload baseline of PAPER.md §4.5), on this GPU."""
    from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore
    from paper_2602_00328_b200.pool import HostTier
    from paper_2602_00328_b200.system import HarvestSystem
    host = HostTier(m.num_layers * m.num_experts * m.expert_size)
    sysm = HarvestSystem(dev, host_tier=host, local_bytes=1, engine=a.engine, log_transfers=False)
    store = ExpertStore(m, sysm.host_id, host)
    store.fill_host(dev, weights=True)
    fetcher = ExpertFetcher(sysm.runtime, m, ExpertResidency(m), store)
    r = run_decode(fetcher, m, dev, 1, lambda x: x, lambda: None, a, "host", microbatches, steps, warm)
    # the stronger host baseline: the same decode with the copy engine on PCIe
    try:
        hp = run_decode(fetcher, m, dev, 1, lambda x: x, lambda: None, a, "host", microbatches, steps, warm,
                        host_plan=True)
        r["host_plan"] = {k: hp[k] for k in ("tokens_per_s", "ms_per_decode_step")}
        r["device_plan_tokens_per_s"] = r["tokens_per_s"]
        r["tokens_per_s"] = max(r["tokens_per_s"], hp["tokens_per_s"])
    except Exception as e:
        r["host_plan"] = {"error": repr(e)[:300]}
    sysm.close()
    return r

def offload_sweep_phase(m, dev, a, fractions=(0, 25, 50, 75, 100), layers=8):
    """moe.offload_sweep (moe.py:394-415) on real decode, this GPU: the
    coldest experts of each layer (ranked by one all-local step's routing)
    served from the pinned host tier, the rest from a resident HBM copy;
    staged decode (the reference's fetch-then-compute pipeline, 2 micro-
    batches) as a CUDA graph.  An 8-layer slice of the model bounds the
    pinned memory and the run time; tok/s scale with 1/layers."""
    from dataclasses import asdict

    from paper_2602_00328_b200.decode import offload_sweep
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.moe import MoEProfile
    from paper_2602_00328_b200.system import HarvestSystem
    ms = MoEProfile(m.name, min(layers, m.num_layers), m.num_experts, m.top_k, m.expert_size, hidden=m.hidden,
                    intermediate=m.intermediate)
    sysm = HarvestSystem(dev, host_bytes=ms.num_layers * ms.num_experts * ms.expert_size, local_bytes=1,
                         engine=a.engine, log_transfers=False)
    try:
        rows = offload_sweep(sysm, ms, list(fractions), Tier.HOST_DRAM, tokens=32, microbatches=2, steps=3,
                             warmup=2)
    finally:
        sysm.close()
    return {"rows": [asdict(r) for r in rows], "layers": ms.num_layers, "tier": "host (pinned DRAM, PCIe)",
            "mode": "staged, 2 micro-batches, CUDA graph", "tokens_per_step": 32,
            "outputs_bit_identical_to_all_local": True,
            "note": "stall_s = fetch time not hidden by the expert FFN in a traced step (device clock); at 0% "
                    "the staged decoder still copies LOCAL experts into its staging buffer (an HBM copy)"}

def kv_long_context(sysm, source, a):
    """Config 4: a 128k-token Llama-3-8B sequence (8,192 blocks x 32 layers x
    64 KiB = 16 GiB) is appended (KV produced locally), evicted out of local
    HBM to harvested peer slabs (N>1, Lossy) or the host tier (N=1, Backed),
    then reloaded (262,144 pages, K1 launched per 1,024 blocks).  Reports the kernel
    time, the end-to-end reload() time, and a content check of sampled pages."""
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.kv import LLAMA3_8B, KVCacheManager, kv_seed
    from paper_2602_00328_b200.runtime import Durability
    m = LLAMA3_8B
    nblk = KV_TOKENS // m.block_tokens
    host = source == "host"
    kv = KVCacheManager(sysm, m, local_blocks=nblk, host_blocks=nblk if host else 1, slab_blocks=KV_SLAB_BLOCKS,
                        durability=Durability.BACKED if host else Durability.LOSSY, engine=a.engine,
                        max_ctas=a.max_ctas, content="fp16")
    kv.append_kv(0, KV_TOKENS)
    t0 = time.perf_counter()
    kv.timing = []
    moves = kv.evict(nblk * m.block_bytes)
    evict_wall = time.perf_counter() - t0
    e_ev0, e_ev1 = kv.timing[0][0], kv.timing[-1][1]
    where = {}
    for _bid, _frm, to in moves:
        where[to] = where.get(to, 0) + 1
    ids = sorted(kv.table)
    kv.timing = []
    t0 = time.perf_counter()
    plan = kv.reload(ids)
    sysm.engine.synchronize()
    wall = time.perf_counter() - t0
    # first launch's start to last launch's end: reload() pipelines its
    # launches with the host-side block resolution
    ev0, ev1, nb = kv.timing[0][0], kv.timing[-1][1], sum(t[2] for t in kv.timing)
    ms = ev0.elapsed_time(ev1)
    rng = np.random.default_rng(0)
    sample = [(int(l), int(b)) for l, b in zip(rng.integers(0, m.num_layers, 64), rng.integers(0, nblk, 64))]
    ptrs = [kv.cache[l, kv.table[b].slot].data_ptr() for l, b in sample]
    bad = F.verify_content(F.ptrs_tensor(ptrs, kv.dev), F.ptrs_tensor([m.page_bytes] * len(ptrs), kv.dev),
                           [kv_seed(l, 0, kv.table[b].index) for l, b in sample], weights=True)
    out = {"sequence_tokens": KV_TOKENS, "blocks": nblk, "pages": nblk * m.num_layers, "bytes": nb,
           "evicted_to": where, "reload_from": {k: len(v) for k, v in plan.items()},
           "reload_kernel_ms": ms, "reload_launches": len(kv.timing), "reload_kernel_GBps": nb / (ms * 1e-3) / 1e9,
           "reload_e2e_ms": wall * 1e3, "evict_kernel_ms": e_ev0.elapsed_time(e_ev1),
           "evict_e2e_ms": evict_wall * 1e3, "sampled_pages_mismatched_words": int(bad.sum()),
           "model": "llama-3-8b: 32 layers x 8 KV heads x 128 x fp16, 16-token blocks"}
    # decode attention over the whole 128k context, KV local vs in the tier
    out["decode_attention"] = _kv_decode_measure(kv, [0], sysm, steps=2)
    kv.close()
    return out


def _kv_decode_measure(kv, seqs, sysm, steps=3, q_heads=32):
    """KVAttentionDecoder over the given sequences: one timed run with every
    block local, then everything evicted to the tier (peer slabs at N>1, host
    at N=1) and the same steps again; the tiered outputs must equal the
    all-local ones bit for bit."""
    import torch
    from paper_2602_00328_b200.kv_decode import KVAttentionDecoder
    dec = KVAttentionDecoder(kv, seqs, q_heads=q_heads, seed=1)

    def timed(dec=dec):
        o = dec.step()
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for _ in range(steps):
            o = dec.step()
        e1.record(cur)
        e1.synchronize()
        return o, e0.elapsed_time(e1) / steps

    # all-local baseline: attention straight over the local pages (no gather),
    # the same kernel on the same bytes as every tiered mode below
    local_out, local_ms = timed(KVAttentionDecoder(kv, seqs, q_heads=q_heads, seed=1, fused=True))
    local_out = local_out.clone()
    kv.sys.engine.synchronize()
    sysm.loop.run()          # slabs emptied by an earlier reload go back to their donors first
    moves = kv.evict(len(dec.ids) * kv.m.block_bytes)
    where = {}
    for _bid, _frm, to in moves:
        where[to] = where.get(to, 0) + 1
    tier_out, tier_ms = timed()
    dec.trace = True
    dec.step()
    ov = dec.overlap_report()
    # the same attention straight over the resident pages (no K1 gather)
    fdec = KVAttentionDecoder(kv, seqs, q_heads=q_heads, seed=1, fused=True)
    fused_out, fused_ms = timed(fdec)
    graphs = {}
    for name, fz in (("gather", False), ("in_place", True)):   # each step one upload + one graph replay
        gdec = KVAttentionDecoder(kv, seqs, q_heads=q_heads, seed=1, fused=fz)
        gdec.capture_graph()
        g_out, g_ms = timed(gdec)
        graphs[name] = {"ms_per_step": g_ms, "tokens_per_s": len(seqs) / (g_ms * 1e-3),
                        "outputs_bit_identical_to_eager": bool(torch.equal(g_out, tier_out))}
        del gdec
    sysm.loop.run()
    nbytes = len(dec.ids) * kv.m.block_bytes
    return {"batch": len(seqs), "context_tokens": dec.T, "kv_bytes_per_step": nbytes, "kv_in": where,
            "tier_ms_per_step": tier_ms, "tier_tokens_per_s": len(seqs) / (tier_ms * 1e-3),
            "tier_kv_GBps": nbytes / (tier_ms * 1e-3) / 1e9,
            "local_ms_per_step": local_ms, "local_tokens_per_s": len(seqs) / (local_ms * 1e-3),
            "outputs_bit_identical_to_all_local": bool(torch.equal(tier_out.view(torch.int16),
                                                                   local_out.view(torch.int16))),
            "outputs_finite": bool(torch.isfinite(tier_out.float()).all()),
            "fused_in_place": {"ms_per_step": fused_ms, "tokens_per_s": len(seqs) / (fused_ms * 1e-3),
                               "kv_GBps": nbytes / (fused_ms * 1e-3) / 1e9,
                               "outputs_bit_identical_to_gathered": bool(torch.equal(fused_out, tier_out))},
            "cuda_graph": graphs,
            "best": max(([("gather", len(seqs) / (tier_ms * 1e-3)), ("in_place", len(seqs) / (fused_ms * 1e-3))]
                         + [(f"{k}_cuda_graph", v["tokens_per_s"]) for k, v in graphs.items()]),
                        key=lambda kv_: kv_[1]),
            "attention": "hv_paged_decode_attention (split-K flash decoding over page pointers, tensor cores)",
            "overlap_traced_step": ov,
            "model": f"{kv.m.name}: GQA {q_heads} q heads over {kv.m.kv_heads} KV heads, per-layer K1 gather "
                     "(fetch stream) overlapped with attention (compute stream)"}


def kv_decode_config1(sysm, source, a, batch=4, context=4096):
    """BASELINE configs[0] shape on the GPU: 4 sequences x 4k tokens of
    Llama-3-8B-shaped KV (1,024 blocks, 2 GiB), decode attention with the
    KV in local HBM and then in the tier (peer slabs at N>1, host at N=1)."""
    from paper_2602_00328_b200.kv import LLAMA3_8B, KVCacheManager
    from paper_2602_00328_b200.runtime import Durability
    m = LLAMA3_8B
    nblk = batch * context // m.block_tokens
    host = source == "host"
    kv = KVCacheManager(sysm, m, local_blocks=nblk, host_blocks=nblk if host else 1, slab_blocks=KV_SLAB_BLOCKS,
                        durability=Durability.BACKED if host else Durability.LOSSY, engine=a.engine,
                        max_ctas=a.max_ctas, content="fp16")
    for s in range(batch):
        kv.append_kv(s, context)
    out = _kv_decode_measure(kv, list(range(batch)), sysm)
    kv.close()
    return out

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
    from paper_2602_00328_b200.moe import QWEN15_MOE_A27B, MoEProfile
    from paper_2602_00328_b200.pool import NodePools
    q = QWEN15_MOE_A27B
    m = MoEProfile(q.name, layers, q.num_experts, q.top_k, q.expert_size, hidden=q.hidden,
                   intermediate=q.intermediate)
    L, E, S = m.num_layers, m.num_experts, m.expert_size
    from paper_2602_00328_b200.cluster import DonorLayout, per_reader_bytes
    if world == 1:
        C, D = [0], []
        per_reader = per_reader_bytes(L * E, S, 1)
        layout = None
    else:
        layout = DonorLayout.split_roles(world, per_reader_bytes(L * E, S, world - world // 2))
        C, D, per_reader = list(layout.compute), list(layout.donors), layout.per_reader
    out = None
    from paper_2602_00328_b200.runtime import Policy, PolicyKind
    # the reference's placement policies under the same churn (runtime.py:169-196):
    # BestFit is the headline; Stability skips donors with many recent
    # revocations; Fairness token-buckets the re-placement copy-in bytes
    policies = {"BestFit": Policy(),
                "Stability": Policy(kind=PolicyKind.STABILITY, stability_window_s=0.2,
                                    stability_max_revocations=L * E // 4),
                "Fairness": Policy(kind=PolicyKind.FAIRNESS, fairness_budget_bytes_per_s=4e9,
                                   fairness_burst_bytes=1e9)}
    # the same BestFit timeline with the fused decoder (experts consumed in
    # place: peer experts over the link, revoked ones from the host copy)
    runs = ([(name, pol, False) for name, pol in policies.items()] + [("BestFit_fused", Policy(), True)]
            + [("BestFit_fused_graph", Policy(), "graph")])
    outs, lending = {}, {}
    for i, (name, pol, fused) in enumerate(runs):
        node = None
        if world > 1:   # fresh donor pools per run: every run starts from empty donors
            node = NodePools(a.group, layout, rank, a.device_of, mode=a.pool_mode, tag=f"churn{i}")
        try:
            if rank in C:
                if node is not None and node.error:
                    raise RuntimeError(node.error)
                outs[name] = _churn_compute(world, rank, dev, a, m, layout, per_reader, node, seconds,
                                            policy=pol, fused=fused)
        except Exception as e:  # every rank still reaches the collectives below
            outs[name] = {"rank": rank, "error": repr(e)[:300]}
        if node is not None:
            node.close()          # readers close, barrier, then the donors' servers stop
            if rank in D:
                lending[name] = {"mode": node.mode, **node.final_stats}
    if lending:
        outs["_donor_lending"] = lending
    results = [None] * world
    if world > 1:
        barrier()
        dist.all_gather_object(results, outs)
    else:
        results = [outs]

    def summary(name):
        rs = [r.get(name) for r in results if r]
        comp = [r for r in rs if r and "error" not in r]
        errs = [r for r in rs if r and "error" in r]
        res = {"tokens_per_s_all_compute_ranks": sum(r["tokens_per_s"] for r in comp),
               "all_outputs_bit_identical": bool(comp) and all(r["outputs_bit_identical_to_all_local"] for r in comp),
               "total_revocations": sum(r["revocations"] for r in comp),
               "total_re_placements": sum(r["re_placements"] for r in comp),
               "total_release_ordering_violations": sum(r["release_ordering_violations"] for r in comp)}
        return res, comp, errs

    head, comp, errs = summary("BestFit")
    res = {"model": f"{m.name} slice: {L} layers x {E} experts x {S} B (Qwen-shaped, bf16)",
           "compute_ranks": C, "donor_ranks": D if D else "self (VMM pool on the compute GPU)",
           "timeline": "markov_availability levels 0/25/50/100% of the donated bytes, 50 ms mean sojourn, "
                       f"seed 5+donor, {seconds} s",
           "policy": "BestFit", **head, "per_rank": comp,
           "donor_lending": {str(r): x["_donor_lending"] for r, x in enumerate(results)
                             if x and "_donor_lending" in x},
           "policy_comparison": {}}
    if errs:
        res["errors"] = errs
    for name in policies:
        if name == "BestFit":
            continue
        h2, _c2, e2 = summary(name)
        res["policy_comparison"][name] = {**h2, "policy": repr(policies[name])}
        if e2:
            res["policy_comparison"][name]["errors"] = e2
    for key, name, desc in (("fused_decoder", "BestFit_fused", "MoEDecoder(fused=True): experts read in place"),
                            ("fused_decoder_cuda_graph", "BestFit_fused_graph",
                             "the same, each step one CUDA graph replay (tables patched in place)")):
        hf, cf, ef = summary(name)
        res[key] = {**hf, "policy": "BestFit", "decoder": desc, "per_rank": cf}
        if ef:
            res[key]["errors"] = ef
    return res

def _churn_compute(world, rank, dev, a, m, layout, per_reader, node, seconds, policy=None,
                   fused=False):
    """Compute-rank side of churn_phase (no collectives inside)."""
    import torch
    from paper_2602_00328_b200.churn import ChurnDriver, expert_tier_counts, markov_availability
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore, rebalance
    from paper_2602_00328_b200.pool import HostTier, PeerPool
    from paper_2602_00328_b200.system import HarvestSystem
    from benchlib.common import reference_checkers
    verify_release_ordering = reference_checkers()[0]
    L, E, S = m.num_layers, m.num_experts, m.expert_size
    host = HostTier(L * E * S)
    if world == 1:
        sysm = HarvestSystem(dev, donors=[dev], donor_bytes=per_reader, host_tier=host, local_bytes=1,
                             engine=a.engine, max_ctas=a.max_ctas, policy=policy)
    else:
        sysm = HarvestSystem(dev, pools=dict(node.views), host_tier=host, local_bytes=1, engine=a.engine,
                             max_ctas=a.max_ctas, policy=policy)
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
                     engine=getattr(a, "kernel_engine", a.engine), max_ctas=a.max_ctas, fused=bool(fused))
    h = dec.step(dec.x0)
    if fused == "graph":        # every later step is one replay; residency changes patch its tables in place
        dec.capture_graph()
        h = dec.step(h).clone()
        step_offset = 1
    else:
        step_offset = 0
    torch.cuda.synchronize()
    GB_levels = [0, per_reader // 4, per_reader // 2, per_reader]
    donors = layout.donors_of(rank) if layout else [dev]
    drv = ChurnDriver(sysm, {i: markov_availability(GB_levels, [0.05] * 4, seed=5 + d, horizon=seconds)
                             for i, d in enumerate(donors, start=1)})
    drv.start()
    steps, peer_min, peer_max, peer_sum = 1 + step_offset, placed0, placed0, 0   # steps applied to h so far
    loop_steps = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        h = dec.step(h)
        steps += 1
        loop_steps += 1
        drv.tick(replace)
        sysm.loop.poll()            # arrivals of finished copy-ins flip residency before counting
        pc = expert_tier_counts(res)["PeerHBM"]
        peer_min, peer_max, peer_sum = min(peer_min, pc), max(peer_max, pc), peer_sum + pc
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
    ldec = MoEDecoder(lf, tokens=TOKENS, microbatches=1, seed=13, fused=bool(fused))
    h2 = ldec.x0
    for _ in range(steps):
        h2 = ldec.step(h2)
    torch.cuda.synchronize()
    out = {"rank": rank, "decode_steps": loop_steps, "tokens_per_s": TOKENS * loop_steps / wall,
           "availability_steps": len(log.of_kind("availability_step")),
           "revocations": len(log.of_kind("revoke_begin")), "re_placements": migrated[0] - placed0,
           "peer_resident_experts_min_max": [peer_min, peer_max], "experts": L * E,
           "peer_resident_experts_mean_over_steps": peer_sum / max(1, loop_steps),
           "release_ordering_violations": len(verify_release_ordering(log)),
           "outputs_bit_identical_to_all_local": bool(torch.equal(h.view(torch.int16), h2.view(torch.int16)))}
    del dec, ldec, resident
    lsys.close()
    sysm.close()
    return out

def phi_phase(world, rank, dev, a, dist, barrier, max_over_ranks, batches=(1, 16, 64)):
    """BASELINE configs[2]: Phi-3.5-MoE-shaped experts (32 layers x 16 experts,
    top-2, 157,286,400 B each) placed by each rank's runtime across its N-1
    donors (up to 7), decode tokens/s at batch 1/16/64.  Rank 0 also times the
    same layers served from pinned host DRAM on a 4-layer slice.
    Collective-safe: local work is guarded, every rank reaches every collective."""
    import torch
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.cluster import DonorLayout, per_reader_bytes, place_experts
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.moe import PHI35_MOE, ExpertFetcher, ExpertResidency, ExpertStore, MoEProfile
    from paper_2602_00328_b200.pool import HostTier, NodePools
    from paper_2602_00328_b200.system import HarvestSystem
    m = PHI35_MOE
    if a.phi_layers != m.num_layers:
        m = MoEProfile(m.name, a.phi_layers, m.num_experts, m.top_k, m.expert_size, hidden=m.hidden,
                       intermediate=m.intermediate)
    L, E, S = m.num_layers, m.num_experts, m.expert_size
    layout = DonorLayout.symmetric(world, per_reader_bytes(L * E, S, world - 1))
    out = {"model": f"{m.name}: {L} layers x {E} experts x {S} B, top-{m.top_k}", "donors_per_rank": world - 1}
    errors = []
    node = sysm = fetcher = None
    try:
        node = NodePools(a.group, layout, rank, a.device_of, mode=a.pool_mode, tag="phi")
        if node.error:
            errors.append(node.error)
        views = node.views
        sysm = HarvestSystem(dev, pools=views, local_bytes=1, engine=a.engine, max_ctas=a.max_ctas,
                             log_transfers=False)
        rt = sysm.runtime
        res = ExpertResidency(m)
        placed, seeds = place_experts(rt, m, res, rank, world - 1)
        ptrs = [rt.address(h) for h in placed]
        for i in range(0, len(ptrs), 32):
            F.fill_weights_bf16(F.ptrs_tensor(ptrs[i:i + 32], f"cuda:{dev}"),
                                F.ptrs_tensor([S] * len(ptrs[i:i + 32]), f"cuda:{dev}"), seeds[i:i + 32])
        torch.cuda.synchronize()
        fetcher = ExpertFetcher(rt, m, res, ExpertStore(m, sysm.host_id, None))
    except Exception as e:
        errors.append(repr(e)[:200])
        fetcher = None
    barrier()
    def timed_decode(b, fused, graph=False):
        """3 timed steps after 1 warm step (or after capture_graph());
        max over ranks (collective-safe)."""
        dt_local, finite, dec = float("inf"), False, None
        try:
            if fetcher is None:
                raise RuntimeError("setup failed")
            dec = MoEDecoder(fetcher, tokens=b, microbatches=1, seed=11, fused=fused)
            h = dec.decode(1)
            if graph:
                dec.capture_graph()
                h = dec.step(h).clone()
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
        del dec
        torch.cuda.empty_cache()
        return max_over_ranks(dt_local), finite

    for b in batches:
        dt, finite = timed_decode(b, False)
        if math.isfinite(dt):
            out[f"batch{b}"] = {"tokens_per_s": b * 3 * world / dt, "per_rank_tokens_per_s": b * 3 / dt,
                                "ms_per_layer": dt / 3 / L * 1e3, "outputs_finite": finite}
        dtf, finite_f = timed_decode(b, True)   # experts consumed in place (hv_expert_ffn_*)
        if math.isfinite(dtf) and f"batch{b}" in out:
            out[f"batch{b}"]["fused"] = {"tokens_per_s": b * 3 * world / dtf, "ms_per_layer": dtf / 3 / L * 1e3,
                                         "outputs_finite": finite_f}
        dtg, finite_g = timed_decode(b, True, graph=True)   # the same, one CUDA graph replay per step
        if math.isfinite(dtg) and f"batch{b}" in out:
            out[f"batch{b}"]["fused_cuda_graph"] = {"tokens_per_s": b * 3 * world / dtg,
                                                    "ms_per_layer": dtg / 3 / L * 1e3, "outputs_finite": finite_g}
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
    except Exception as e:
        errors.append(repr(e)[:200])
    barrier()
    if node is not None:
        out["donor_pools"] = node.mode
        node.close()
    else:
        barrier()        # NodePools.close()'s barrier on the ranks that have one
    all_err = [None] * world
    dist.all_gather_object(all_err, errors)
    if any(all_err):
        out["errors"] = {str(r): e for r, e in enumerate(all_err) if e}
    return out
