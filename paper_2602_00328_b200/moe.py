"""MoE expert offload over the Harvest runtime: residency, placement, and the
per-stage expert fetch hook.

Reference: moe.py.  Kept API: MoEProfile/MoEModelSpec (profiles.py:79-86),
PipelineConfig (moe.py:40-48), RoutingTrace (:51-62), expert_content
(:114-115), ResidencyEntry/ExpertResidency (:118-152), rebalance (:155-197),
place_offloaded (:354-383).  The fetch hook _DecodeRun._issue_fetches
(:282-313) — one app_transfer per activated non-local expert — becomes
``ExpertFetcher.issue_fetches``: the same per-expert tier decision
(LOCAL skip / live PEER handle / HOST authoritative copy) but ONE launch of the
K2 batched-fetch kernel for the whole stage, issued on the fetch stream one
stage ahead of compute, with the drain tracked per touched handle.

Expert bytes are real: the authoritative copy of expert (layer, e) sits in the
pinned host tier at ``ExpertStore.host_offset(layer, e)`` and holds the
synthetic content keyed by expert_content() (splitmix64 stream, see
oracle/hv_oracle.c); peers hold copies made by the placement copy-in (K3).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import fetch as F
from ._nvtx import annotate
from .memalloc import Segment, Tier
from .runtime import AllocationHints, Durability, HarvestHandle, HarvestRuntime, stable_hash64


@dataclass(frozen=True)
class MoEProfile:
    """profiles.py:79-86, plus the dense shapes needed to run the FFN."""
    name: str
    num_layers: int
    num_experts: int
    top_k: int
    expert_size: int
    compute_time_per_microbatch: float = 0.0
    hidden: int = 0
    intermediate: int = 0


MoEModelSpec = MoEProfile

# BASELINE.json configs[1] and [2]; bf16 gate+up+down = 3*hidden*inter*2 bytes
QWEN15_MOE_A27B = MoEProfile("qwen1.5-moe-a2.7b", num_layers=24, num_experts=60, top_k=4,
                             expert_size=3 * 2048 * 1408 * 2, hidden=2048, intermediate=1408)
PHI35_MOE = MoEProfile("phi-3.5-moe", num_layers=32, num_experts=16, top_k=2,
                       expert_size=3 * 4096 * 6400 * 2, hidden=4096, intermediate=6400)
assert QWEN15_MOE_A27B.expert_size == 17_301_504 and PHI35_MOE.expert_size == 157_286_400


@dataclass
class PipelineConfig:
    """moe.py:40-48."""
    microbatch_tokens: int = 324
    num_microbatches: int = 14
    local_cache_experts: int = 0

    def validate(self) -> None:
        if self.microbatch_tokens <= 0 or self.num_microbatches <= 0:
            raise ValueError("pipeline counts must be positive")


@dataclass
class RoutingTrace:
    """moe.py:51-62: active[microbatch][layer] = sorted expert ids."""
    num_microbatches: int
    num_layers: int
    num_experts: int
    active: list
    counts: np.ndarray

    def active_set(self, microbatch: int, layer: int) -> tuple[int, ...]:
        return self.active[microbatch][layer]


def expert_content(model: MoEProfile, layer: int, expert: int) -> int:
    """moe.py:114-115 — also the seed of the expert's synthetic bytes."""
    return stable_hash64("expert", model.name, layer, expert)


def topk_routing(model: MoEProfile, tokens: int, steps: int, seed: int) -> list[list[np.ndarray]]:
    """Router top-k over N(0,1) logits per token (decode batch ``tokens``):
    routing[step][layer] = sorted unique activated experts."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(steps):
        row = []
        for _layer in range(model.num_layers):
            logits = rng.standard_normal((tokens, model.num_experts))
            top = np.argpartition(-logits, model.top_k - 1, axis=1)[:, :model.top_k]
            row.append(np.unique(top))
        out.append(row)
    return out


@dataclass
class ResidencyEntry:
    tier: Tier
    handle: HarvestHandle | None = None


class ExpertResidency:
    """moe.py:124-152; every expert keeps its authoritative host copy."""

    def __init__(self, model: MoEProfile):
        self.model = model
        self.entries: dict[tuple[int, int], ResidencyEntry] = {
            (layer, e): ResidencyEntry(Tier.HOST_DRAM) for layer in range(model.num_layers)
            for e in range(model.num_experts)}
        self._listeners = []

    def get(self, layer: int, expert: int) -> ResidencyEntry:
        return self.entries[(layer, expert)]

    def set_tier(self, layer: int, expert: int, tier: Tier, handle: HarvestHandle | None = None) -> None:
        self.entries[(layer, expert)] = ResidencyEntry(tier, handle)
        for fn in self._listeners:
            fn(layer, expert, tier, handle)

    def on_change(self, fn) -> None:
        self._listeners.append(fn)

    def on_tier(self, tier: Tier) -> list[tuple[int, int]]:
        return [key for key, e in self.entries.items() if e.tier == tier]

    def content_hashes(self) -> dict[tuple[int, int], int]:
        return {key: expert_content(self.model, *key) for key in self.entries}


class ExpertStore:
    """Host-authoritative expert bytes: expert (layer, e) at offset
    ``(layer * E + e) * expert_size`` of the host tier (device id host_id)."""

    def __init__(self, model: MoEProfile, host_device_id: int, host_tier=None, base_offset: int = 0):
        self.model = model
        self.host_device_id = host_device_id
        self.host = host_tier
        self.base_offset = base_offset
        # byte layout of every copy of an expert: "row" (gate [I][H], up [I][H],
        # down [H][I], row-major) or "tiled" (the same matrices as HV_FFN_TILED
        # swizzled 128 x 64 tiles, for the tcgen05 K4's bulk-copy weight stream)
        self.layout = "row"

    def host_offset(self, layer: int, expert: int) -> int:
        return self.base_offset + (layer * self.model.num_experts + expert) * self.model.expert_size

    def host_segment(self, layer: int, expert: int) -> Segment:
        return Segment(self.host_offset(layer, expert), self.model.expert_size)

    def fill_host(self, device: int = 0, layers=None, weights: bool = False, layout: str = "row") -> None:
        """Write every expert's synthetic content into the pinned host tier
        (the fill kernel writes through the mapped alias over PCIe).
        ``weights=True`` writes the bf16-weights variant (finite values).
        ``layout="tiled"`` then stores each matrix of those logical weights as
        HV_FFN_TILED tiles (fetch.tile_expert_matrix); every later copy of the
        expert (peer, staging) carries the same bytes."""
        m = self.model
        if layout not in ("row", "tiled"):
            raise ValueError(f"unknown expert layout {layout!r}")
        if layout == "tiled" and not weights:
            raise ValueError("the tiled layout is a layout of bf16 weights (weights=True)")
        if layout == "tiled" and (m.hidden % 128 or m.intermediate % 128):
            raise ValueError("tiled experts need hidden and intermediate sizes that are multiples of 128")
        layers = range(m.num_layers) if layers is None else layers
        fill = F.fill_weights_bf16 if weights else F.fill_content
        for layer in layers:
            ptrs = [self.host.device_address(self.host_offset(layer, e)) for e in range(m.num_experts)]
            fill(F.ptrs_tensor(ptrs, f"cuda:{device}"), F.ptrs_tensor([m.expert_size] * m.num_experts, f"cuda:{device}"),
                 [expert_content(m, layer, e) for e in range(m.num_experts)])
        torch.cuda.synchronize(device)
        if layout == "tiled":
            view = self.host.view()
            H, I = m.hidden, m.intermediate
            for layer in layers:
                for e in range(m.num_experts):
                    o = self.host_offset(layer, e)
                    cpu = torch.from_numpy(view[o:o + m.expert_size])          # aliases the pinned host tier
                    w = cpu.to(f"cuda:{device}").view(torch.bfloat16)
                    t = torch.cat([F.tile_expert_matrix(w[:I * H].view(I, H)).reshape(-1),
                                   F.tile_expert_matrix(w[I * H:2 * I * H].view(I, H)).reshape(-1),
                                   F.tile_expert_matrix(w[2 * I * H:].view(H, I)).reshape(-1)])
                    cpu.copy_(t.view(torch.uint8))
            torch.cuda.synchronize(device)
        self.layout = layout

    def host_digests(self, device: int = 0) -> np.ndarray:
        """Digest of every expert's authoritative host copy ([L, E] uint64,
        hv_digest over the mapped host tier): the expected values of the
        per-fetch content check (ExpertFetcher.enable_content_check)."""
        m = self.model
        out = np.empty((m.num_layers, m.num_experts), dtype=np.uint64)
        sizes = F.ptrs_tensor([m.expert_size] * m.num_experts, f"cuda:{device}")
        for layer in range(m.num_layers):
            ptrs = [self.host.device_address(self.host_offset(layer, e)) for e in range(m.num_experts)]
            d = F.digest(F.ptrs_tensor(ptrs, f"cuda:{device}"), sizes)
            out[layer] = d.cpu().numpy().view(np.uint64)
        return out


def rebalance(sim, runtime: HarvestRuntime, model: MoEProfile, residency: ExpertResidency,
              counts: np.ndarray, host_device_id: int, max_migrations: int | None = None,
              store: ExpertStore | None = None) -> list[tuple[int, int, HarvestHandle]]:
    """moe.py:155-197: hottest host-resident experts -> harvest_alloc (Backed,
    client "moe") -> callback -> host->peer copy-in; residency flips to PEER
    on arrival iff the handle is still live; stops at the first NoCapacity.
    All copy-ins of one call go out as one batched launch (K3)."""
    store = store or ExpertStore(model, host_device_id)
    candidates = list(residency.on_tier(Tier.HOST_DRAM))
    candidates.sort(key=lambda le: (-int(counts[le[0], le[1]]), le))
    migrations, items = [], []
    for layer, expert in candidates:
        if max_migrations is not None and len(migrations) >= max_migrations:
            break
        handle = runtime.harvest_alloc(model.expert_size,
                                       AllocationHints(durability=Durability.BACKED, client_id="moe"))
        if handle is None:
            break
        tag = ("expert", layer, expert)
        runtime.set_tag(handle, tag)

        def _revoked(h, reason, layer=layer, expert=expert):
            residency.set_tier(layer, expert, Tier.HOST_DRAM, None)

        runtime.harvest_register_cb(handle, _revoked)

        def _arrived(xfer, content, layer=layer, expert=expert, h=handle):
            if runtime.is_live(h):
                residency.set_tier(layer, expert, Tier.PEER_HBM, h)

        items.append(dict(src=(host_device_id, store.host_segment(layer, expert)),
                          dst=(handle.device_id, Segment(handle.base, handle.size)),
                          size=model.expert_size, tag=tag, handle=handle,
                          payload=expert_content(model, layer, expert), on_complete=_arrived))
        migrations.append((layer, expert, handle))
    if items:
        runtime.app_transfer_batch(items, engine=getattr(runtime, "placement_engine", None))
    return migrations


def place_offloaded(sim, runtime: HarvestRuntime, model: MoEProfile, residency: ExpertResidency,
                    trace: RoutingTrace, fraction_pct: float, tier: Tier, host_device_id: int,
                    store: ExpertStore | None = None) -> None:
    """moe.py:354-383: pin the hottest experts locally, offload the coldest
    fraction per layer to ``tier`` (peer placement falls back to host)."""
    if not 0 <= fraction_pct <= 100:
        raise ValueError("fraction must be within [0, 100]")
    n = model.num_experts
    n_off = int(round(n * fraction_pct / 100.0))
    offloaded = []
    for layer in range(model.num_layers):
        order = sorted(range(n), key=lambda e: (int(trace.counts[layer, e]), e))
        for e in order[:n_off]:
            residency.set_tier(layer, e, Tier.HOST_DRAM)
            offloaded.append((layer, e))
        for e in order[n_off:]:
            residency.set_tier(layer, e, Tier.LOCAL_HBM)
    if tier == Tier.PEER_HBM and offloaded:
        rebalance(sim, runtime, model, residency, trace.counts, host_device_id,
                  max_migrations=len(offloaded), store=store)
        sim.run()
    elif tier not in (Tier.PEER_HBM, Tier.HOST_DRAM):
        raise ValueError(f"offload tier must be peer or host, got {tier}")


class ExpertFetcher:
    """Batched stage fetch hook (replaces _DecodeRun._issue_fetches, moe.py:282-313).

    ``issue_fetches(layer, experts, dst_ptrs)`` resolves each expert's serving
    tier exactly as the reference does — LOCAL: skipped; PEER with a live
    handle: read from the donor (the handle joins the batch's drain set);
    otherwise: read the host-authoritative copy — and moves all of them with
    one K2 launch.  Returns the FetchBatch (plan + completion event).
    """

    def __init__(self, runtime: HarvestRuntime, model: MoEProfile, residency: ExpertResidency,
                 store: ExpertStore, local_addr=None):
        self.rt = runtime
        self.model = model
        self.residency = residency
        self.store = store
        self.engine = runtime.engine
        L, E = model.num_layers, model.num_experts
        host_base = runtime.engine.memory.base(store.host_device_id) if store.host is not None else 0
        # per-expert source address tables; kept in sync by residency listeners
        self.host_addr = np.array([[host_base + store.host_offset(l, e) for e in range(E)] for l in range(L)],
                                  dtype=np.uint64)
        self.src_addr = self.host_addr.copy()
        # device addresses of locally resident expert weights (LOCAL tier); the
        # fetch plan skips them exactly like moe.py:295-296
        self.local_addr = (np.zeros((L, E), dtype=np.uint64) if local_addr is None
                           else np.asarray(local_addr, dtype=np.uint64).reshape(L, E))
        self.tier = np.full((L, E), 2, dtype=np.int8)   # 0 local, 1 peer, 2 host
        self.handles: dict[tuple[int, int], HarvestHandle] = {}
        for (l, e), ent in residency.entries.items():
            self._update(l, e, ent.tier, ent.handle)
        residency.on_change(self._update)
        self.sizes_cache: dict[int, np.ndarray] = {}
        self.expected = None   # [L, E] digests of the authoritative copies (enable_content_check)
        self.reads = 0         # DecodeMetrics.reads (moe.py:200-208): objects fetched

    def enable_content_check(self, expected_digests: np.ndarray, stream=None) -> None:
        """Check the content identity of every fetch, as the reference does on
        every arrival (moe.py:315-319: ``content != expected`` -> read_errors):
        after each stage's fetch, hv_check_digests_batch digests what arrived
        on ``stream`` (default: a new stream of the fetch device) and counts
        the objects whose digest differs from ``expected_digests[layer, e]``.
        The check runs beside the next stage's fetch; ``FetchBatch.event`` then
        covers the fetch and its check (reuse the staging buffer after it)."""
        L, E = self.model.num_layers, self.model.num_experts
        exp = np.ascontiguousarray(expected_digests, dtype=np.uint64)
        if exp.shape != (L, E):
            raise ValueError(f"expected digests must be [{L}, {E}]")
        dev = self.engine.cuda_device
        self.expected = exp
        self._check_stream = N.stream_handle(stream) if stream is not None else self._new_stream(dev)
        self._scratch = torch.zeros(E, dtype=torch.int64, device=f"cuda:{dev}")
        self._flags = torch.zeros(E, dtype=torch.uint8, device=f"cuda:{dev}")
        self._errors = torch.zeros(1, dtype=torch.int64, device=f"cuda:{dev}")
        self._fscratch = torch.zeros(E, dtype=torch.int64, device=f"cuda:{dev}")   # fused (fetch-stream) path
        self._fflags = torch.zeros(E, dtype=torch.uint8, device=f"cuda:{dev}")
        self._last_flags = self._flags
        self._check_events = []
        self.fetches_checked = 0

    @staticmethod
    def _new_stream(dev: int) -> int:
        import ctypes as C
        s = C.c_void_p()
        N.call("hv_stream_create", dev, 0, C.byref(s))
        return s.value or 0

    def read_errors(self) -> int:
        """DecodeMetrics.read_errors (moe.py:200-208): fetched objects whose
        bytes differed from their authoritative copy, over every checked
        stage so far (synchronizes the check stream)."""
        if self.expected is None:
            raise RuntimeError("content check not enabled (enable_content_check)")
        N.call("hv_stream_synchronize", self._check_stream)
        self.engine.synchronize()
        return int(self._errors.cpu().item())

    def last_read_error_flags(self) -> np.ndarray:
        """Per-object mismatch flags of the most recent checked stage."""
        N.call("hv_stream_synchronize", self._check_stream)
        self.engine.synchronize()
        return self._last_flags.cpu().numpy()

    def _update(self, layer, expert, tier, handle) -> None:
        self.version = getattr(self, "version", 0) + 1
        if tier == Tier.LOCAL_HBM:
            self.tier[layer, expert] = 0
            self.handles.pop((layer, expert), None)
        elif tier == Tier.PEER_HBM and handle is not None:
            self.tier[layer, expert] = 1
            self.handles[(layer, expert)] = handle
            self.src_addr[layer, expert] = self.rt.address(handle)
        else:
            self.tier[layer, expert] = 2
            self.handles.pop((layer, expert), None)
            self.src_addr[layer, expert] = self.host_addr[layer, expert]

    def plan(self, layer: int, experts) -> list[tuple[int, str]]:
        """Per-expert serving tier, in the reference's order (moe.py:290-313)."""
        out = []
        for e in experts:
            t = self.tier[layer, e]
            if t == 0:
                continue
            h = self.handles.get((layer, int(e)))
            out.append((int(e), "peer" if (t == 1 and h is not None and self.rt.is_live(h)) else "host"))
        return out

    @annotate("harvest.issue_fetches")
    def issue_fetches(self, layer: int, experts, dst_ptrs) -> "FetchBatch":
        experts = np.asarray(experts, dtype=np.int64)
        dst_ptrs = np.asarray(dst_ptrs, dtype=np.uint64)
        t = self.tier[layer, experts]
        keep = t != 0
        ex, dst = experts[keep], dst_ptrs[keep]
        peer_mask = t[keep] == 1
        handles = []
        if peer_mask.any():
            for e in ex[peer_mask]:
                h = self.handles[(layer, int(e))]
                if self.rt.is_live(h):
                    handles.append(h)
                else:  # invalidated between table update and now: host copy
                    self.tier[layer, e] = 2
                    self.src_addr[layer, e] = self.host_addr[layer, e]
        src = np.ascontiguousarray(self.src_addr[layer, ex])
        n = len(ex)
        sizes = self.sizes_cache.get(n)
        if sizes is None:
            sizes = self.sizes_cache[n] = np.full(n, self.model.expert_size, dtype=np.uint64)
        batch = self.rt.begin_reads(handles) if handles else None
        event = None
        self.reads += n
        if n:
            cbs = [lambda _x, b=batch: self.rt.end_reads(b)] if batch else []
            dst = np.ascontiguousarray(dst)
            if self.expected is not None and peer_mask.any():
                # peer experts: the SM kernel copies and digests them in one
                # pass (hv_swap_blocks_batch_checked); host-tier ones ride the
                # copy engine and are digested after it, inside the same call
                exp = np.ascontiguousarray(self.expected[layer, ex])
                self.engine.launch_raw_checked(src, dst, sizes, exp, self._fscratch.data_ptr(),
                                               self._fflags.data_ptr(), self._errors.data_ptr(), callbacks=cbs)
                self._last_flags = self._fflags
                event = self.engine.last_event
            else:
                self.engine.launch_raw(src, dst, sizes, callbacks=cbs)
                event = self.engine.last_event
                if self.expected is not None:
                    event = self._check(layer, ex, dst, sizes, event)
                    self._last_flags = self._flags
        return FetchBatch(layer, ex, t[keep].copy(), event)

    def _check(self, layer, ex, dst, sizes, fetch_event):
        """Digest the stage's arrivals on the check stream (after the fetch)
        and count mismatches against the authoritative digests."""
        import ctypes as C
        N.call("hv_stream_wait_event", self._check_stream, fetch_event)
        exp = np.ascontiguousarray(self.expected[layer, ex])
        N.call("hv_check_digests_batch", dst.ctypes.data, sizes.ctypes.data, exp.ctypes.data, len(ex),
               self._scratch.data_ptr(), self._flags.data_ptr(), self._errors.data_ptr(), self._check_stream)
        # a small ring of check events (the fetch engine recycles its own)
        if len(self._check_events) < 8:
            e = C.c_void_p()
            N.call("hv_event_create", self.engine.cuda_device, 0, C.byref(e))
            self._check_events.append(e)
        ev = self._check_events[self.fetches_checked % len(self._check_events)]
        N.call("hv_event_record", ev, self._check_stream)
        self.fetches_checked += 1
        return ev


@dataclass
class FetchBatch:
    layer: int
    experts: np.ndarray
    tiers: np.ndarray
    event: object

    def wait_on(self, stream) -> None:
        """Make ``stream`` (e.g. the compute stream) wait for this stage's fetch.
        Call before the runtime's loop polls the batch (events are recycled)."""
        if self.event is not None:
            N.call("hv_stream_wait_event", N.stream_handle(stream), self.event)
