"""CPU legs of the benchmark: the oracle port timed on host cores (cpu_baseline, --impl reference).

Test infrastructure use of oracle/ is confined to this module, as the contract allows."""
from __future__ import annotations

import os
import sys
import time

import numpy as np

from benchlib.common import METRIC, emit, routing, shape, workload_config


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

def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_nexp(m, host_buf):
    return (host_buf.size // m.expert_size) if isinstance(host_buf, np.ndarray) else m.num_layers * m.num_experts

def cpu_host_copy(m, n_experts):
    """A host-resident expert table for the CPU legs (content from the oracle)."""
    from oracle import harvest_oracle as O
    buf = np.empty(n_experts * m.expert_size, dtype=np.uint8)
    O.fill_batch([buf.ctypes.data + i * m.expert_size for i in range(n_experts)], [m.expert_size] * n_experts,
                 [O.expert_seed(m.name, i // m.num_experts, i % m.num_experts) for i in range(n_experts)],
                 threads=os.cpu_count() or 1)
    return buf

def run_reference(a):
    """--impl reference: the reference CPU path of the fetch (the oracle port:
    a memcpy gather of every layer's activated experts from the
    host-authoritative expert table) on all host cores, rank 0 only.

    Same workload as the B200 arm: the full 24-layer x 60-expert table
    (24.9 GB of host memory, content from the oracle's generator), the same
    routing, every layer of every step, the same --steps/--warmup.  This
    process never imports paper_2602_00328_b200: the only native library it
    maps is oracle/build/libhv_oracle.so."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import harvest_oracle as O
    m = shape()
    threads = os.cpu_count() or 1
    host = cpu_host_copy(m, m.num_layers * m.num_experts)
    routes = routing(m, a.steps + a.warmup)
    dst = np.empty(m.num_experts * m.expert_size, dtype=np.uint8)
    dst[::4096] = 0   # fault the destination in before timing
    dp_all = [dst.ctypes.data + i * m.expert_size for i in range(m.num_experts)]

    def one_step(step):
        moved = 0
        t0 = time.perf_counter()
        for layer, ex in enumerate(step):
            src = [host.ctypes.data + (layer * m.num_experts + int(e)) * m.expert_size for e in ex]
            O.gather(src, dp_all[:len(ex)], [m.expert_size] * len(ex), threads=threads)
            moved += len(ex) * m.expert_size
        return moved, time.perf_counter() - t0

    for s in range(a.warmup):
        one_step(routes[s])
    moved = dt = 0.0
    for s in range(a.warmup, a.warmup + a.steps):
        mv, t = one_step(routes[s])
        moved += mv
        dt += t
    gbps = moved / dt / 1e9
    line = {"metric": METRIC, "value": gbps, "unit": "GB/s", "impl": "reference", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * dt / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic", "config": workload_config(m, a.gpus),
            "implementation": {"source_tier": "host DRAM (the reference CPU path: memcpy gather of the "
                                              "host-authoritative expert table on rank 0)", "threads": threads},
            "cpu_baseline": {"value": gbps, "unit": "GB/s", "cores": threads, "kind": "port", "cpu_model": cpu_model(),
                             "sample": f"every layer ({m.num_layers}) of every decode step, memcpy gather from a "
                                       f"{m.num_layers * m.num_experts * m.expert_size / 1e9:.1f} GB host expert "
                                       f"table (oracle/hv_oracle.c, {threads} threads)"},
            "e2e": {"value": gbps, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    try:
        line["reference_simulator"] = reference_simulator(m, max(0, a.gpus - 1))
    except Exception as e:
        line["reference_simulator"] = {"error": repr(e)[:300]}
    emit(line, a)
    return 0


def reference_simulator(m, n_peers: int, steps: int = 4) -> dict:
    """The reference's own fetch path, unmodified, timed on one host core:
    ``harvestsim.moe.simulate_decode`` (moe.py:343-351) with the workload's
    model shape, every expert offloaded (moe.py:354-383) to the host tier
    (n_peers == 0) or placed on n_peers modeled peers.  It moves no bytes: the
    result is its Python cost per ``app_transfer`` (runtime.py:320-364) and
    the decode rate its calibrated model (profiles.py:51-57, H100) predicts.
    Imported from the pip-installed copy under baseline/_ref (never from
    /root/reference, which does not exist on the GPU box)."""
    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "harvestsim")):
        return {"unavailable": "baseline/_ref/harvestsim not installed"}
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from harvestsim import moe as RM, profiles as RP
    from harvestsim.events import Simulator
    from harvestsim.memalloc import Tier
    from harvestsim.runtime import HarvestRuntime
    prof = RP.MoEProfile(m.name, num_layers=m.num_layers, num_experts=m.num_experts, top_k=m.top_k,
                         expert_size=m.expert_size, compute_time_per_microbatch=0.0)
    pipe = RM.PipelineConfig(microbatch_tokens=32, num_microbatches=steps)
    trace = RM.generate_routing(prof, pipe, 0.0, 0, 2)  # skew 0 = uniform routing, as bench's N(0,1) logits
    sim = Simulator()
    topo = RP.build_topology(RP.PAPER_H100, num_peers=n_peers)
    rt = HarvestRuntime(sim, topo)
    host_id = topo.devices[-1].device_id
    res = RM.ExpertResidency(prof)
    t0 = time.perf_counter()
    RM.place_offloaded(sim, rt, prof, res, trace, 100.0, Tier.PEER_HBM if n_peers else Tier.HOST_DRAM, host_id)
    t_place = time.perf_counter() - t0
    t0 = time.perf_counter()
    met = RM.simulate_decode(sim, rt, prof, pipe, trace, res, host_id)
    wall = time.perf_counter() - t0
    moved = met.reads * m.expert_size
    return {"impl": "harvestsim (reference, unmodified, baseline/_ref)", "cores": 1,
            "tier": "peer" if n_peers else "host", "modeled_peers": n_peers, "decode_steps": steps,
            "fetches": met.reads, "read_errors": met.read_errors,
            "wall_s": wall, "wall_us_per_fetch": 1e6 * wall / max(1, met.reads),
            "placement_wall_s": t_place,
            "modeled_decode_s": met.decode_time, "modeled_tok_s": met.tokens_per_s,
            "modeled_GBps": moved / met.decode_time / 1e9 if met.decode_time > 0 else None,
            "note": "simulator: moves no bytes; modeled numbers use its H100 calibration (55 GB/s host, "
                    "495 GB/s peer) with zero compute time, so they are link-model predictions"}
