"""CPU legs of the benchmark: the oracle port timed on host cores (cpu_baseline, --impl reference).

Test infrastructure use of oracle/ is confined to this module, as the contract allows."""
from __future__ import annotations

import json
import math
import os
import statistics
import sys
import time

import numpy as np

from benchlib.common import METRIC, emit, model, routing, workload_config


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
