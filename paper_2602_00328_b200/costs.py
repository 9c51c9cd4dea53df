"""Measured costs for the KV fallback decision.

``resolve_fallback`` picks FetchFromHost iff the host transfer of a block is
no slower than recomputing its entries.  The reference states both sides as
model constants: the host link (fixed_cost, bandwidth) of its calibration
profile (profiles.py:58-64) and ``recompute_time_per_entry`` (a default of
1 s that makes recompute never win).  On B200 both are measured:

* ``measure_host_link``: K1/K2 fetch latency from the pinned host tier into
  local HBM over a range of block sizes, refit with the reference's own
  least-squares ``calibrate`` (interconnect.py:168-188) into a LinkSpec;
* ``measure_recompute``: the time to regenerate the KV of ``e`` entries --
  a chunked prefill of ``e`` tokens through every layer of the model's
  dense shape (QKV projection, causal attention over the chunk, output
  projection, gated MLP; bf16 on cuBLAS / SDPA flash, random weights, one
  CUDA graph per chunk size), which is what recomputing a lost block costs
  the serving engine.  Attention over an earlier prefix and launch overhead
  are not included, so this is a lower bound on recompute.

``RecomputeCost`` holds the measured curve (entries -> seconds, linear
interpolation, extrapolated at the measured large-chunk rate), and
``fallback_crossover`` solves the decision boundary on it.
"""
from __future__ import annotations

import bisect
from dataclasses import dataclass, field

import numpy as np
import torch

from .interconnect import LinkKind, LinkSpec, calibrate, calibration_rms, transfer_time


@dataclass(frozen=True)
class DenseShape:
    """The transformer shape whose prefill regenerates the KV cache."""
    name: str
    num_layers: int
    hidden: int
    q_heads: int
    kv_heads: int
    head_dim: int
    intermediate: int


LLAMA3_8B_DENSE = DenseShape("llama-3-8b", num_layers=32, hidden=4096, q_heads=32, kv_heads=8, head_dim=128,
                             intermediate=14336)


@dataclass
class RecomputeCost:
    """Measured recompute time of ``e`` KV entries (seconds), from points
    (entries, seconds) sorted by entries."""
    points: list = field(default_factory=list)

    def __call__(self, entries: int) -> float:
        if entries <= 0:
            return 0.0
        xs = [p[0] for p in self.points]
        i = bisect.bisect_left(xs, entries)
        if i < len(xs) and xs[i] == entries:
            return self.points[i][1]
        if i == 0:                          # below the smallest chunk: no cheaper than it
            return self.points[0][1]
        if i == len(xs):                    # beyond: the largest chunk's per-entry rate
            e, t = self.points[-1]
            return t * entries / e
        (e0, t0), (e1, t1) = self.points[i - 1], self.points[i]
        return t0 + (t1 - t0) * (entries - e0) / (e1 - e0)

    @property
    def per_entry_rate(self) -> float:
        """Asymptotic seconds per entry (the largest measured chunk)."""
        e, t = self.points[-1]
        return t / e


def fetch_wins(link: LinkSpec, entries: int, bytes_per_entry: int, recompute) -> bool:
    """FetchFromHost iff transfer_time(block bytes) <= recompute
    time; ``recompute`` is seconds per entry (the SPEC's linear form) or a
    callable entries -> seconds (a measured curve)."""
    t_host = transfer_time(link, entries * bytes_per_entry)
    t_rec = recompute(entries) if callable(recompute) else entries * recompute
    return t_host <= t_rec


def fallback_crossover(link: LinkSpec, bytes_per_entry: int, recompute, max_entries: int = 1 << 16) -> dict:
    """Where the decision flips in 1..max_entries.  For the linear form the
    SPEC's closed form alpha + e*b/B = e*r gives e* = alpha / (r - b/B)
    (SPEC.md:425); the scan is exact for either form."""
    out = {"max_entries": max_entries}
    if not callable(recompute):
        slope = recompute - bytes_per_entry / link.bandwidth
        out["closed_form_e_star"] = link.fixed_cost / slope if slope > 0 else None
    decisions = [fetch_wins(link, e, bytes_per_entry, recompute) for e in (1, max_entries)]
    flips = []
    prev = fetch_wins(link, 1, bytes_per_entry, recompute)
    # the decision is monotone for the linear form; scan coarsely, then refine
    e, step = 1, 1
    while e < max_entries:
        nxt = min(max_entries, e + step)
        cur = fetch_wins(link, nxt, bytes_per_entry, recompute)
        if cur != prev:
            lo, hi = e, nxt
            while hi - lo > 1:
                mid = (lo + hi) // 2
                if fetch_wins(link, mid, bytes_per_entry, recompute) == prev:
                    lo = mid
                else:
                    hi = mid
            flips.append({"last_entries_" + ("fetch" if prev else "recompute"): lo,
                          "first_entries_" + ("fetch" if cur else "recompute"): hi})
            prev = cur
            e = hi
            step = 1
            continue
        e = nxt
        step = min(step * 2, 4096)
    out["decision_at_1"] = "FetchFromHost" if decisions[0] else "Recompute"
    out["decision_at_max"] = "FetchFromHost" if decisions[1] else "Recompute"
    out["flips"] = flips
    return out


def measure_host_link(host_tier, device: int = 0, sizes=(65536, 262144, 1 << 20, 4 << 20, 16 << 20),
                      engine: str = "auto", iters: int = 5) -> tuple[LinkSpec, dict]:
    """Fetch latency from the pinned host tier into local HBM (one object
    of each size through the library's engine per source), refit with
    calibrate().  Returns the LinkSpec and the measured points."""
    from . import _native as N
    nbytes = max(sizes)
    if host_tier.nbytes < nbytes:
        raise ValueError("host tier smaller than the largest calibration size")
    dst = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
    s = torch.cuda.Stream(device=f"cuda:{device}")
    src = np.array([host_tier.device_address(0)], dtype=np.uint64)
    d = np.array([dst.data_ptr()], dtype=np.uint64)
    pts = []
    for nb in sizes:
        z = np.array([nb], dtype=np.uint64)
        ts = []
        for i in range(iters + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            N.call("hv_swap_blocks_batch", src.ctypes.data, d.ctypes.data, z.ctypes.data, 1, N.ENGINES[engine], 0,
                   s.cuda_stream)
            e1.record(s)
            e1.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1) * 1e-3)
        pts.append((nb, float(np.median(ts))))
    fc, bw = calibrate(pts)
    link = LinkSpec(LinkKind.HOST_LINK, fc, bw, endpoints=(0, -1))
    return link, {"points_us": [[n, t * 1e6] for n, t in pts], "fixed_cost_us": fc * 1e6,
                  "bandwidth_GBps": bw / 1e9, "rms_rel": calibration_rms(pts, fc, bw)}


def measure_recompute(shape: DenseShape = LLAMA3_8B_DENSE, chunks=(16, 64, 256, 1024, 4096), device: int = 0,
                      iters: int = 3, seed: int = 0) -> RecomputeCost:
    """Time a chunked prefill of ``e`` tokens through ``shape.num_layers``
    layers (distinct random bf16 weights per layer, so the weight stream is
    real), for each chunk size; returns the (entries, seconds) curve."""
    dev = torch.device(f"cuda:{device}")
    g = torch.Generator(device=dev).manual_seed(seed)
    H, I, D = shape.hidden, shape.intermediate, shape.head_dim
    q_out, kv_out = shape.q_heads * D, shape.kv_heads * D
    std = H ** -0.5

    def w(*dims):
        return (torch.randn(*dims, device=dev, dtype=torch.bfloat16, generator=g) * std)

    layers = [dict(qkv=w(H, q_out + 2 * kv_out), o=w(q_out, H), gu=w(H, 2 * I), down=w(I, H) * (H / I) ** 0.5)
              for _ in range(shape.num_layers)]
    rep = shape.q_heads // shape.kv_heads

    def forward(x):
        T = x.shape[0]
        for p in layers:
            qkv = x @ p["qkv"]
            q = qkv[:, :q_out].view(T, shape.q_heads, D).transpose(0, 1)
            k = qkv[:, q_out:q_out + kv_out].view(T, shape.kv_heads, D).transpose(0, 1)
            v = qkv[:, q_out + kv_out:].view(T, shape.kv_heads, D).transpose(0, 1)
            if rep > 1:   # grouped-query heads expanded so SDPA takes its fused (flash) kernel
                k = k.repeat_interleave(rep, dim=0)
                v = v.repeat_interleave(rep, dim=0)
            a = torch.nn.functional.scaled_dot_product_attention(q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0),
                                                                 is_causal=True)[0]
            x = x + a.transpose(0, 1).reshape(T, q_out) @ p["o"]
            gu = x @ p["gu"]
            x = x + (torch.nn.functional.silu(gu[:, :I]) * gu[:, I:]) @ p["down"]
        return x

    # device time of the prefill, captured as one CUDA graph per chunk size so
    # the per-op launch cost of eager PyTorch (~300 ops) does not count: a
    # lower bound on what recomputing the entries costs a serving engine
    pts = []
    with torch.no_grad():
        for T in chunks:
            x = torch.randn(T, H, device=dev, dtype=torch.bfloat16, generator=g)
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                for _ in range(2):
                    forward(x)
            torch.cuda.current_stream(dev).wait_stream(side)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                forward(x)
            ts = []
            for i in range(iters + 1):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                graph.replay()
                e1.record()
                e1.synchronize()
                if i:
                    ts.append(e0.elapsed_time(e1) * 1e-3)
            pts.append((int(T), float(np.median(ts))))
            del graph
    del layers
    torch.cuda.empty_cache()
    return RecomputeCost(sorted(pts))
