"""KV-cache offload over Harvest: block table, append/evict/reload, revocation
fallback, and the block-table-indexed page gather (K1).

The reference ships no KV code; its contract is SPEC.md:367-460 (module
``kv_sim``): BlockTable (:380-383), OffloadPolicy (:384-387), append_kv
(:390-398), evict (:399-407), reload (:408-416), resolve_fallback (:417-425),
reload_latency_experiment (:426-434); defaults: 16-token blocks (:444), Lossy
durability (:447).  PAPER.md §5.2 (lines 308-314) describes the vLLM
integration it models (KVOffloadManager + OffloadingHandler).

B200 layout.  A page is one layer of one 16-token block, K and V:
``block_tokens * kv_heads * head_dim * 2 * dtype_bytes`` (Llama-3-8B: 65,536 B).
Every tier stores pages layer-major, ``[layer][slot]``, like vLLM's per-layer
KV tensors, so page (l, b) of block b lives at ``base[b] + l * stride[b]``:

  local HBM   base = cache + slot*page        stride = local_blocks*page
  peer slab   base = slab_va + slot*page      stride = slab_blocks*page
  host tier   base = host_alias + slot*page   stride = host_blocks*page

Peer memory is taken in slabs of ``slab_blocks`` blocks through
``harvest_alloc`` (one revocable handle per slab, not per 64 KiB page); a slab
revocation invalidates its blocks: Backed blocks fall back to their host copy,
Lossy blocks become NotMaterialized (recompute).  The data movement of an
evict/reload call (all pages of all blocks, all layers) is K1
(``hv_kv_gather_blocks``) over four per-block arrays (source base/stride,
destination base/stride) resolved from the table on the host, launched every
``launch_chunk_blocks`` blocks so the device copies one chunk while the host
resolves the next; the per-layer gather resolves one pointer per page.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import fetch as F
from ._nvtx import annotate
from .interconnect import LinkSpec, transfer_time
from .pool import HostTier
from .runtime import AllocationHints, Durability, HarvestHandle, RevokeReason, StaleHandleError, stable_hash64


class KVTier(enum.Enum):
    LOCAL_HBM = "LocalHBM"
    PEER_HBM = "PeerHBM"
    HOST_DRAM = "HostDRAM"
    NOT_MATERIALIZED = "NotMaterialized"


_T = {KVTier.LOCAL_HBM: 0, KVTier.PEER_HBM: 1, KVTier.HOST_DRAM: 2, KVTier.NOT_MATERIALIZED: 3}


class TierExhausted(Exception):
    """Neither the peer tier nor the host tier can hold a block."""


@dataclass(frozen=True)
class KVModelSpec:
    """SPEC.md:372-375 plus the dense shape that defines a page."""
    name: str
    num_layers: int
    kv_heads: int
    head_dim: int
    dtype_bytes: int = 2
    block_tokens: int = 16
    recompute_time_per_entry: float = 1.0

    @property
    def page_bytes(self) -> int:
        return self.block_tokens * self.kv_heads * self.head_dim * 2 * self.dtype_bytes

    @property
    def bytes_per_entry(self) -> int:
        return self.num_layers * self.kv_heads * self.head_dim * 2 * self.dtype_bytes

    @property
    def block_bytes(self) -> int:
        return self.num_layers * self.page_bytes


LLAMA3_8B = KVModelSpec("llama-3-8b", num_layers=32, kv_heads=8, head_dim=128)
assert LLAMA3_8B.page_bytes == 65536 and LLAMA3_8B.bytes_per_entry == 131072


class EvictionOrder(enum.Enum):
    LRU = "LRU"
    FIFO = "FIFO"
    SEQUENCE_TAIL = "SequenceTail"


@dataclass
class OffloadPolicy:
    """SPEC.md:384-387."""
    order: EvictionOrder = EvictionOrder.LRU
    local_watermark: float = 1.0

    def validate(self) -> None:
        if not 0.0 < self.local_watermark <= 1.0:
            raise ValueError("watermark must be in (0, 1]")


# Residency version: bumped by every change of where a block's pages are
# (tier, slot, slab, host slot) or of a slab's mapping, so a reader that caches
# a resolved page table (kv_decode) re-resolves exactly when it must.  Tracked
# at the attribute level, so no mutation path can skip it.
_residency = [0]
_RESIDENCY_FIELDS = frozenset(("tier", "slot", "slab", "host_slot", "va", "live", "handle"))


def residency_version() -> int:
    return _residency[0]


class _Tracked:
    def __setattr__(self, name, value):
        if name in _RESIDENCY_FIELDS:
            _residency[0] += 1
        object.__setattr__(self, name, value)


@dataclass
class KVBlock(_Tracked):
    """SPEC.md:376-383 (one BlockTable entry)."""
    block_id: int
    sequence_id: int
    index: int
    entries: int
    durability: Durability
    tier: KVTier = KVTier.LOCAL_HBM
    slot: int = -1                 # local slot, peer slab slot, or host slot
    slab: int = -1                 # peer slab index when PEER_HBM
    host_slot: int | None = None   # authoritative host copy (Backed, or host-resident)
    last_access: float = 0.0
    created: int = 0


def kv_seed(layer: int, seq: int, block_index: int) -> int:
    """Content identity of page (layer, seq, block) — stable_hash64 of its tag."""
    return stable_hash64("kv", layer, seq, block_index)


@dataclass
class _Slab(_Tracked):
    handle: HarvestHandle
    va: int
    free: list = field(default_factory=list)
    blocks: dict = field(default_factory=dict)  # slot -> block_id
    live: bool = True


class KVCacheManager:
    """Block table + offloading handler for one compute GPU (a HarvestSystem)."""

    def __init__(self, system, model: KVModelSpec, local_blocks: int, host_blocks: int,
                 policy: OffloadPolicy | None = None, slab_blocks: int = 32,
                 durability: Durability = Durability.LOSSY, engine: str = "auto", max_ctas: int = 0,
                 spread: bool = True, content: str = "raw"):
        self.sys = system
        self.spread = spread
        # page content: "raw" splitmix bytes, or "fp16" -- the same keyed stream
        # with every 16-bit lane mapped to a finite fp16 value (+-[1, 1.125)),
        # for consumers that compute on the KV (kv_decode)
        if content not in ("raw", "fp16"):
            raise ValueError("content must be 'raw' or 'fp16'")
        self.content = content
        self.rt = system.runtime
        self.m = model
        self.policy = policy or OffloadPolicy()
        self.policy.validate()
        self.default_durability = durability
        self.engine = N.ENGINES[engine]
        self.max_ctas = max_ctas
        self.dev = f"cuda:{system.compute}"
        self.page = model.page_bytes
        self.L = model.num_layers
        self.local_blocks, self.host_blocks, self.slab_blocks = local_blocks, host_blocks, slab_blocks
        self.cache = torch.empty((self.L, local_blocks, self.page), dtype=torch.uint8, device=self.dev)
        self.host = HostTier(max(1, host_blocks) * self.L * self.page)
        self.local_free = list(range(local_blocks - 1, -1, -1))
        self.host_free = list(range(host_blocks - 1, -1, -1))
        self.table: dict[int, KVBlock] = {}
        self.slabs: list[_Slab] = []
        self.seq_blocks: dict[int, list[int]] = {}
        self._next_id = 0
        self._created = 0
        self.stream = system.engine.stream
        # reload() launches K1 every this many resolved blocks (1,024 Llama-3-8B
        # blocks = 2 GiB, ~2.7 ms over NVLink: far above launch cost, while
        # the host resolves the next chunk)
        self.launch_chunk_blocks = 1024
        # block moves whose blocks are consecutive in source and destination go
        # out as per-layer runs through the engine per source (F.layer_runs)
        self.coalesce = True
        self.recomputed = 0
        self.stats = {"evict_peer": 0, "evict_host": 0, "reload_peer": 0, "reload_host": 0, "recompute": 0}

    # ------------------------------------------------------------ addressing
    def _page_base(self, b: KVBlock) -> tuple[int, int]:
        if b.tier == KVTier.LOCAL_HBM:
            return self.cache.data_ptr() + b.slot * self.page, self.local_blocks * self.page
        if b.tier == KVTier.PEER_HBM:
            return self.slabs[b.slab].va + b.slot * self.page, self.slab_blocks * self.page
        if b.tier == KVTier.HOST_DRAM:
            return self.host.device_address(b.host_slot * self.page), self.host_blocks * self.page
        raise ValueError(f"block {b.block_id} is not materialized")

    def _host_base(self, host_slot: int) -> tuple[int, int]:
        return self.host.device_address(host_slot * self.page), self.host_blocks * self.page

    def _launch_blocks(self, src_b, src_s, dst_b, dst_s, handles=(), on_done=None) -> None:
        """One K1 launch (hv_kv_gather_blocks) moving every layer of each
        listed block: page (l, b) from src_b[b] + l*src_s[b] to dst_b[b] +
        l*dst_s[b].  Only the four per-block arrays are uploaded (pinned,
        stream-ordered on the fetch stream); drain tracked on `handles`."""
        n = len(src_b)
        if n == 0:
            if on_done:
                on_done()
            return
        runs = F.layer_runs(src_b, src_s, dst_b, dst_s, self.page, self.L) if self.coalesce else None
        if runs is not None:
            # consecutive slots (a sequence evicted together): a few long
            # per-layer runs through the engine per source -- the copy engine
            # when they come from the pinned host tier
            batch = self.rt.begin_reads(list(handles)) if handles else None

            def _done_runs(_x, batch=batch):
                if batch is not None:
                    self.rt.end_reads(batch)
                if on_done:
                    on_done()

            timing = getattr(self, "timing", None)
            if timing is not None:
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record(torch.cuda.ExternalStream(self.stream, device=self.dev))
            src, dst, nbytes = runs
            N.call("hv_swap_blocks_batch", src.ctypes.data, dst.ctypes.data, nbytes.ctypes.data, len(src),
                   self.engine, self.max_ctas, self.stream)
            if timing is not None:
                ev1.record(torch.cuda.ExternalStream(self.stream, device=self.dev))
                timing.append((ev0, ev1, int(nbytes.sum())))
            self.sys.engine.track([_done_runs])
            return
        arrs = [np.ascontiguousarray(x, dtype=np.uint64) for x in (src_b, src_s, dst_b, dst_s)]
        batch = self.rt.begin_reads(list(handles)) if handles else None

        def _done(_x, batch=batch):
            if batch is not None:
                self.rt.end_reads(batch)
            if on_done:
                on_done()

        timing = getattr(self, "timing", None)
        if timing is not None:  # kernel-only time of this launch, on the fetch stream
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(torch.cuda.ExternalStream(self.stream, device=self.dev))
        # the four per-block arrays go through the library's pinned ring (an SM
        # kernel uploads them: no DMA queued behind copy-engine traffic)
        N.call("hv_kv_gather_blocks_h", arrs[0].ctypes.data, arrs[1].ctypes.data, arrs[2].ctypes.data,
               arrs[3].ctypes.data, n, self.L, self.page, self.engine, self.max_ctas, self.stream)
        self.sys.engine.track([_done])
        if timing is not None:
            ev1.record(torch.cuda.ExternalStream(self.stream, device=self.dev))
            timing.append((ev0, ev1, n * self.L * self.page))

    # ------------------------------------------------------------ append
    def append_kv(self, sequence_id: int, tokens: int, durability: Durability | None = None) -> list[int]:
        """Fill the sequence's open tail block, then new LocalHBM blocks; new
        pages get their content (the KV the decode step produced)."""
        if tokens <= 0:
            raise ValueError("tokens must be > 0")
        dur = durability or self.default_durability
        blocks = self.seq_blocks.setdefault(sequence_id, [])
        touched = []
        now = self.sys.loop.now
        self._pending_fill = []
        while tokens > 0:
            tail = self.table[blocks[-1]] if blocks else None
            if tail is not None and tail.entries < self.m.block_tokens:
                if tail.tier != KVTier.LOCAL_HBM:
                    self.reload([tail.block_id])
                take = min(tokens, self.m.block_tokens - tail.entries)
                tail.entries += take
                if tail.host_slot is not None:
                    # the host copy predates these entries: drop it, so the
                    # next evict writes a fresh one instead of serving a stale
                    # page after a fallback.  Reads of the slot
                    # already enqueued precede any later write on the stream.
                    self.host_free.append(tail.host_slot)
                    tail.host_slot = None
                tail.last_access = now
                tokens -= take
                touched.append(tail.block_id)
                continue
            slot = self._take_local_slot()
            bid = self._next_id
            self._next_id += 1
            self._created += 1
            take = min(tokens, self.m.block_tokens)
            b = KVBlock(bid, sequence_id, len(blocks), take, dur, KVTier.LOCAL_HBM, slot=slot, last_access=now,
                        created=self._created)
            self.table[bid] = b
            blocks.append(bid)
            tokens -= take
            touched.append(bid)
            self._pending_fill.append(b)
        self._flush_fill()
        return touched

    def _flush_fill(self) -> None:
        """Materialize the content of blocks created since the last flush (one
        fill launch); must run before any of them can be evicted."""
        pend = getattr(self, "_pending_fill", None)
        if pend:
            self._pending_fill = []
            self._materialize(pend)

    def _materialize(self, blocks: list[KVBlock]) -> None:
        """Write the blocks' synthetic KV content into their local slots."""
        if not blocks:
            return
        ptrs, seeds = [], []
        for b in blocks:
            base, stride = self._page_base(b)
            for layer in range(self.L):
                ptrs.append(base + layer * stride)
                seeds.append(kv_seed(layer, b.sequence_id, b.index))
        from . import fetch as F
        torch.cuda.synchronize(self.sys.compute)  # slots may be targets of pending copies
        fill = F.fill_weights_bf16 if self.content == "fp16" else F.fill_content
        fill(F.ptrs_tensor(ptrs, self.dev), F.ptrs_tensor([self.page] * len(ptrs), self.dev), seeds)
        torch.cuda.synchronize(self.sys.compute)

    def _local_used(self) -> int:
        return self.local_blocks - len(self.local_free)

    def _take_local_slot(self) -> int:
        limit = int(self.policy.local_watermark * self.local_blocks)
        if self._local_used() + 1 > limit or not self.local_free:
            self._flush_fill()
            self.evict(self.m.block_bytes * max(1, self._local_used() + 1 - limit))
        if not self.local_free:
            raise TierExhausted("local HBM has no free KV slot after eviction")
        return self.local_free.pop()

    # ------------------------------------------------------------ evict
    def _eviction_order(self) -> list[KVBlock]:
        local = [b for b in self.table.values() if b.tier == KVTier.LOCAL_HBM]
        if self.policy.order == EvictionOrder.LRU:
            local.sort(key=lambda b: (b.last_access, b.created))
        elif self.policy.order == EvictionOrder.FIFO:
            local.sort(key=lambda b: b.created)
        else:  # sequence tail: the newest blocks of each sequence first
            local.sort(key=lambda b: (-b.index, b.sequence_id))
        return local

    def _peer_slot(self, durability: Durability) -> tuple[int, int] | None:
        cur = getattr(self, "_open_slab", 0)
        if cur < len(self.slabs) and self._writable(self.slabs[cur]):
            return cur, self.slabs[cur].free.pop()
        for i, s in enumerate(self.slabs):
            if self._writable(s):
                self._open_slab = i
                return i, s.free.pop()
        peers = [st.spec.device_id for st in self.rt.peer_states()]
        # round-robin preference over donors (runtime.py:205-214 hint): a big
        # reload then reads every donor's NVLink egress at once
        pref = [peers[len(self.slabs) % len(peers)]] if (self.spread and peers) else None
        h = self.rt.harvest_alloc(self.slab_blocks * self.L * self.page,
                                  AllocationHints(preferred_devices=pref, durability=durability, client_id="kv"))
        if h is None:
            return None
        idx = len(self.slabs)
        slab = _Slab(h, self.rt.address(h), free=list(range(self.slab_blocks - 1, -1, -1)))
        self.slabs.append(slab)
        self._open_slab = idx
        self.rt.set_tag(h, ("kv-slab", idx))
        self.rt.harvest_register_cb(h, lambda hh, reason, idx=idx: self._on_revoke(idx, reason))
        return idx, slab.free.pop()

    @annotate("harvest.kv_evict")
    def evict(self, bytes_needed: int) -> list[tuple[int, str, str]]:
        """Move LRU/FIFO/tail blocks out of local HBM: to a peer slab when one can
        be harvested (Backed blocks also keep a host copy), else to host.
        The page copies go out as K1 launches of launch_chunk_blocks blocks."""
        if bytes_needed <= 0:
            raise ValueError("bytes_needed must be > 0")
        n_blocks = -(-bytes_needed // self.m.block_bytes)
        victims = self._eviction_order()[:n_blocks]
        moves, src_b, src_s, dst_b, dst_s, handles = [], [], [], [], [], set()
        page, cache0 = self.page, self.cache.data_ptr()
        local_stride, slab_stride = self.local_blocks * page, self.slab_blocks * page
        host0, host_stride = self.host.device_address(0), self.host_blocks * page
        LOCAL, PEER, HOST, BACKED = KVTier.LOCAL_HBM, KVTier.PEER_HBM, KVTier.HOST_DRAM, Durability.BACKED
        to_peer, to_host = [], []
        slab = None
        chunk = max(1, int(self.launch_chunk_blocks))
        launched = 0
        err = None
        try:
            for b in victims:
                sbase = cache0 + b.slot * page
                # fast path: the open slab still has room (else _peer_slot harvests)
                if slab is not None and self._writable(slab):
                    slab_i, slot = cur, slab.free.pop()
                    placed = True
                else:
                    placed = self._peer_slot(b.durability)
                    if placed is not None:
                        cur, slot = placed
                        slab_i, slab = cur, self.slabs[cur]
                if placed is not None:
                    new_host = None
                    if b.durability is BACKED and b.host_slot is None:
                        try:
                            new_host = self._take_host_slot()
                        except TierExhausted:
                            slab.free.append(slot)   # this victim stays local: return its slab slot
                            raise
                    src_b.append(sbase), src_s.append(local_stride)
                    dst_b.append(slab.va + slot * page), dst_s.append(slab_stride)
                    handles.add(slab.handle)
                    if new_host is not None:
                        b.host_slot = new_host
                        src_b.append(sbase), src_s.append(local_stride)
                        dst_b.append(host0 + b.host_slot * page), dst_s.append(host_stride)
                    self.local_free.append(b.slot)
                    b.tier, b.slab, b.slot = PEER, slab_i, slot
                    slab.blocks[slot] = b.block_id
                    to_peer.append(b.block_id)
                else:
                    slab = None
                    if b.host_slot is None:
                        b.host_slot = self._take_host_slot()   # raises before this victim changes
                        src_b.append(sbase), src_s.append(local_stride)
                        dst_b.append(host0 + b.host_slot * page), dst_s.append(host_stride)
                    self.local_free.append(b.slot)
                    b.tier, b.slot = HOST, b.host_slot
                    to_host.append(b.block_id)
                moves.append((b.block_id, "LocalHBM", "PeerHBM" if placed is not None else "HostDRAM"))
                if len(src_b) - launched >= chunk:  # pipelined as in reload()
                    self._launch_blocks(src_b[launched:], src_s[launched:], dst_b[launched:], dst_s[launched:],
                                        handles)
                    launched, handles = len(src_b), set()
        except TierExhausted as e:
            # the victims moved so far keep their new tiers: their copies are
            # launched and drained below before the error propagates, so no
            # table entry ever points at a page that was not written
            err = e
        self.stats["evict_peer"] += len(to_peer)
        self.stats["evict_host"] += len(to_host)
        # one log record per destination tier and call (block ids in order)
        if to_peer:
            self.sys.loop.record("kv_evict", blocks=to_peer, to="PeerHBM")
        if to_host:
            self.sys.loop.record("kv_evict", blocks=to_host, to="HostDRAM")
        if len(src_b) > launched:
            self._launch_blocks(src_b[launched:], src_s[launched:], dst_b[launched:], dst_s[launched:], handles)
        if src_b:
            # freed local slots are reusable only after the copies drained them
            self.sys.engine.synchronize()
            self.sys.loop.poll()
        if err is not None:
            raise err
        return moves

    def _take_host_slot(self) -> int:
        if not self.host_free:
            raise TierExhausted("host tier is full")
        return self.host_free.pop()

    # ------------------------------------------------------------ revocation
    def _on_revoke(self, slab_i: int, reason: RevokeReason) -> None:
        """Slab revoked (runtime.py:403-405 ordering: already drained and
        invalidated): Backed blocks fall back to host, Lossy ones are lost."""
        slab = self.slabs[slab_i]
        slab.live = False
        for slot, bid in list(slab.blocks.items()):
            b = self.table[bid]
            if b.host_slot is not None:
                b.tier, b.slot, b.slab = KVTier.HOST_DRAM, b.host_slot, -1
            else:
                b.tier, b.slot, b.slab = KVTier.NOT_MATERIALIZED, -1, -1
        slab.blocks.clear()
        slab.free = []

    # ------------------------------------------------------------ reload
    def resolve_fallback(self, block: KVBlock, host_link: LinkSpec | None = None) -> str:
        """Backed -> FetchFromHost iff host transfer_time <=
        entries * recompute_time_per_entry, else Recompute; no host copy -> Recompute."""
        if block.host_slot is None:
            return "Recompute"
        link = host_link or getattr(self, "host_link", None) or self.sys.topology.link_between(0, self.sys.host_id)
        rec = getattr(self, "recompute", None)
        if rec is None:
            rec = self.m.recompute_time_per_entry
        t_host = transfer_time(link, block.entries * self.m.bytes_per_entry)
        t_rec = rec(block.entries) if callable(rec) else block.entries * rec
        return "FetchFromHost" if t_host <= t_rec else "Recompute"

    def set_costs(self, host_link: LinkSpec | None = None, recompute=None) -> None:
        """Base resolve_fallback on measured costs (costs.measure_host_link /
        costs.measure_recompute): ``host_link`` replaces the topology's
        constant host link, ``recompute`` the model's recompute_time_per_entry
        (seconds per entry, or a callable entries -> seconds)."""
        if host_link is not None:
            self.host_link = host_link
        if recompute is not None:
            self.recompute = recompute

    @annotate("harvest.kv_reload")
    def reload(self, block_ids) -> dict:
        """Bring blocks to LocalHBM from their resident tier (K1, one launch per
        launch_chunk_blocks resolved blocks, pipelined with the resolution).
        Revoked-peer blocks resolve through resolve_fallback; Lossy blocks
        without a host copy are recomputed (content regenerated)."""
        table, LOCAL, PEER, HOST, NM = self.table, KVTier.LOCAL_HBM, KVTier.PEER_HBM, KVTier.HOST_DRAM, \
            KVTier.NOT_MATERIALIZED
        need = [table[i] for i in block_ids if table[i].tier is not LOCAL]
        plan = {"peer": [], "host": [], "recompute": []}
        recompute, vacated = [], []
        now = self.sys.loop.now
        n = len(need)
        # reserve every destination slot first: evictions triggered here only
        # see blocks that are already local, never the ones being reloaded
        limit = int(self.policy.local_watermark * self.local_blocks)
        if n and len(self.local_free) >= n and self._local_used() + n <= limit:
            # bulk: no eviction needed; ascending slots keep consecutive
            # blocks contiguous in the cache, so the move coalesces into runs
            slots = sorted(self.local_free[-n:])
            del self.local_free[-n:]
        else:
            slots = [self._take_local_slot() for _ in need]
        src_b = np.empty(n, dtype=np.uint64)
        src_s = np.empty(n, dtype=np.uint64)
        dst_b = np.empty(n, dtype=np.uint64)
        k = 0
        page, cache0 = self.page, self.cache.data_ptr()
        slab_stride, host_stride = self.slab_blocks * page, self.host_blocks * page
        host0 = self.host.device_address(0)
        live_cache: dict[int, bool] = {}
        plan_peer, plan_host = plan["peer"], plan["host"]
        dst_s = np.full(n, self.local_blocks * page, dtype=np.uint64)
        # launch every `chunk` resolved blocks: the device copies chunk j while
        # the host resolves chunk j+1, so only the first chunk's resolution
        # shows in the reload latency
        chunk = max(1, int(self.launch_chunk_blocks))
        launched, chunk_handles = 0, set()
        for b, slot in zip(need, slots):
            t = b.tier
            if t is PEER:
                live = live_cache.get(b.slab)
                if live is None:
                    live = live_cache[b.slab] = self.rt.is_live(self.slabs[b.slab].handle)
                if not live:  # revoked between lookup and issue: fallback
                    t = b.tier = HOST if b.host_slot is not None else NM
            if t is HOST and self.resolve_fallback(b) == "Recompute":
                t = b.tier = NM
            if t is NM:
                b.tier, b.slot = LOCAL, slot
                recompute.append(b)
                plan["recompute"].append(b.block_id)
                continue
            if t is PEER:
                slab = self.slabs[b.slab]
                src_b[k], src_s[k] = slab.va + b.slot * page, slab_stride
                chunk_handles.add(slab.handle)
                plan_peer.append(b.block_id)
                vacated.append((b.slab, b.slot))
            else:
                src_b[k], src_s[k] = host0 + b.host_slot * page, host_stride
                plan_host.append(b.block_id)
            dst_b[k] = cache0 + slot * page
            k += 1
            b.tier, b.slot, b.slab = LOCAL, slot, -1
            b.last_access = now
            if k - launched >= chunk:
                self._launch_blocks(src_b[launched:k], src_s[launched:k], dst_b[launched:k], dst_s[launched:k],
                                    chunk_handles)
                launched, chunk_handles = k, set()
        self.stats["recompute"] += len(plan["recompute"])
        self.stats["reload_peer"] += len(plan_peer)
        self.stats["reload_host"] += len(plan_host)
        if k > launched:
            self._launch_blocks(src_b[launched:k], src_s[launched:k], dst_b[launched:k], dst_s[launched:k],
                                chunk_handles)
        # old peer slots become reusable only now: any later write into them is
        # stream-ordered after this launch's reads (same fetch stream)
        for slab_i, slot in vacated:
            slab = self.slabs[slab_i]
            slab.blocks.pop(slot, None)
            if slab.live:
                slab.free.append(slot)
        if recompute:
            self.sys.engine.synchronize()
            self._materialize(recompute)
        self._release_empty_slabs()
        return plan

    def _writable(self, s: _Slab) -> bool:
        """A slab can take new blocks while it has free slots and no release of
        its handle has begun (a revoking slab is being drained; writing into it
        would only extend the drain and lose the block at the callback)."""
        return s.live and bool(s.free) and not self.rt.is_draining(s.handle)

    def _release_empty_slabs(self) -> None:
        for s in self.slabs:
            if s.live and not s.blocks and len(s.free) == self.slab_blocks:
                if self.rt.is_draining(s.handle):
                    continue                 # a revoke is already releasing it; its callback marks it dead
                s.live = False
                self.rt.harvest_free(s.handle)

    # ------------------------------------------------------------ the per-layer gather (C1)
    @annotate("harvest.kv_gather_layer")
    def gather_layer(self, layer: int, block_ids, dst: torch.Tensor, stream=None) -> None:
        """K1: page `layer` of every listed block -> dst[i] (contiguous), read
        from wherever the block is resident (local / peer / host).  The peer
        slabs read join the drain set until the gather completes."""
        bases, strides, handles = self.page_table(block_ids)
        src = bases + np.uint64(layer) * strides
        s = N.stream_handle(stream) if stream is not None else self.stream
        pinned, d_src = self._stage_u64(src, s)   # async, stream-ordered: no host stall
        batch = self.rt.begin_reads(handles) if handles else None
        from . import fetch as F
        F.kv_gather(d_src, self.page, dst=dst, engine=self.engine, max_ctas=self.max_ctas, stream=s)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.ExternalStream(s, device=self.dev))
        if batch is not None:                     # drain: released when the gather is done
            if s != self.stream:
                N.call("hv_stream_wait_event", self.stream, ev.cuda_event)
            self.sys.engine.track([lambda _x, b=batch: self.rt.end_reads(b)])
        self._staged.append((ev, pinned, d_src))   # alive until the gather that reads them is done

    def page_table(self, block_ids) -> tuple[np.ndarray, np.ndarray, list]:
        """Where every listed block's pages are right now: page (l, b) is at
        base[b] + l * stride[b] in the block's resident tier (local, peer slab
        or host).  Also returns the live peer-slab handles those pages are read
        from, for the reader's drain set.  Blocks must be materialized."""
        n = len(block_ids)
        bases = np.empty(n, dtype=np.uint64)
        strides = np.empty(n, dtype=np.uint64)
        handles = {}
        for i, bid in enumerate(block_ids):
            b = self.table[bid]
            bases[i], strides[i] = self._page_base(b)
            if b.tier == KVTier.PEER_HBM:
                h = self.slabs[b.slab].handle
                handles[h.key()] = h
        return bases, strides, list(handles.values())

    def _stage_u64(self, arr: np.ndarray, stream: int) -> tuple[torch.Tensor, torch.Tensor]:
        """Upload a host u64 array through pinned memory on `stream`; the
        caller keeps both buffers referenced until its consumer completes."""
        from collections import deque
        keep = self.__dict__.setdefault("_staged", deque())
        while keep and keep[0][0].query():
            keep.popleft()
        pinned = torch.from_numpy(arr.view(np.int64)).pin_memory()
        with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=self.dev)):   # the writer's pool
            dev = torch.empty(pinned.numel(), dtype=torch.int64, device=self.dev)
        N.call("hv_memcpy_h2d", dev.data_ptr(), pinned.data_ptr(), pinned.numel() * 8, stream)
        return pinned, dev

    def block_pages_local(self, bid: int) -> torch.Tensor:
        b = self.table[bid]
        assert b.tier == KVTier.LOCAL_HBM
        return self.cache[:, b.slot, :]

    def close(self) -> None:
        """Give every harvested slab back to its donor (freed once drained) and
        release the host tier."""
        self.sys.engine.synchronize()
        for s in self.slabs:
            if s.live:
                s.live = False
                try:
                    self.rt.harvest_free(s.handle)
                except StaleHandleError:   # already revoking or released: the runtime finishes it
                    pass
        self.sys.loop.run()
        self.host.close()


def reload_latency_experiment(models, entry_counts, host_link: LinkSpec, peer_link: LinkSpec) -> list[tuple]:
    """modeled host vs peer reload latency and speedup per
    (model, entries) — the prediction side; bench/measure_kv.py measures it."""
    rows = []
    for m in models:
        for e in entry_counts:
            h = transfer_time(host_link, e * m.bytes_per_entry)
            p = transfer_time(peer_link, e * m.bytes_per_entry)
            rows.append((m.name, e, h, p, h / p))
    return rows
