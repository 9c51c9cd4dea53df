"""vLLM KV-offload "PEER" medium backed by harvested peer HBM: both halves.

PAPER.md §5.2 (lines 308-314) extends vLLM's KV manager with a
KVOffloadManager (scheduler side) and a per-device OffloadingHandler (worker
side).  vLLM 0.22's contracts (vllm/v1/kv_offload/):
* ``OffloadingSpec`` (base.py:338-): built by name through
  ``OffloadingSpecFactory.create_spec`` (factory.py:35-58) from
  ``kv_connector_extra_config["spec_name"]``; ``get_manager()`` and
  ``get_handlers(kv_caches)``.  ``HarvestOffloadingSpec`` is registered under
  the name "HarvestOffloadingSpec" (``register_with_vllm``, run at import).
* ``OffloadingManager`` (base.py:110-237): lookup / prepare_load / touch /
  complete_load / prepare_store / complete_store / take_events.
  ``HarvestOffloadingManager`` keeps an LRU of offloaded block keys over a
  fixed id space of peer blocks; a block whose slab was revoked turns into a
  lookup MISS (and a removed event), so vLLM recomputes it -- the Lossy
  semantics of SPEC.md:417-425.
* ``OffloadingHandler`` (worker/worker.py:26-75): transfer_async(job_id,
  (src_spec, dst_spec)) -> bool, get_finished(), wait(job_ids).
  ``HarvestPeerHandler`` moves GPU <-> PEER blocks with the library's fetch
  engines (one launch per job over every page of every KV tensor); a load
  that touches a revoked block completes with success=False.
Peer blocks live in harvested slabs (``PeerBlockPool``): one revocable
Lossy handle per slab of ``slab_blocks`` blocks.
vLLM is imported lazily; without it, minimal stand-ins of its types keep the
adapter importable and testable.
"""
from __future__ import annotations

import time
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .runtime import AllocationHints, Durability, HarvestRuntime

try:  # vLLM >= 0.22 layout
    from vllm.v1.kv_offload.worker.worker import OffloadingHandler, TransferResult  # type: ignore
    from vllm.v1.kv_offload.base import (LoadStoreSpec, OffloadingEvent, OffloadingManager,  # type: ignore
                                         OffloadingSpec, PrepareStoreOutput)
    HAVE_VLLM = True
except Exception:  # pragma: no cover - exercised when vLLM is absent
    HAVE_VLLM = False

    class OffloadingHandler:  # minimal stand-ins
        pass

    class OffloadingManager:
        pass

    class OffloadingSpec:
        def __init__(self, vllm_config, kv_cache_config):
            self.vllm_config, self.kv_cache_config = vllm_config, kv_cache_config
            self.extra_config = vllm_config.kv_transfer_config.kv_connector_extra_config
            self.block_size_factor = 1

    @dataclass
    class TransferResult:
        job_id: int
        success: bool
        transfer_size: int | None = None
        transfer_time: float | None = None
        transfer_type: tuple | None = None

    @dataclass
    class PrepareStoreOutput:
        keys_to_store: list
        store_spec: object
        evicted_keys: list

    @dataclass
    class OffloadingEvent:
        keys: list
        medium: str
        removed: bool

    class LoadStoreSpec:
        pass


class GPUBlocks(LoadStoreSpec):
    """Block ids of the GPU KV cache (vLLM's GPULoadStoreSpec analogue)."""

    def __init__(self, block_ids):
        self.block_ids = np.asarray(block_ids, dtype=np.int64)

    @staticmethod
    def medium() -> str:
        return "GPU"


class PeerBlocks(LoadStoreSpec):
    """Block ids of the harvested peer tier."""

    def __init__(self, block_ids):
        self.block_ids = np.asarray(block_ids, dtype=np.int64)

    @staticmethod
    def medium() -> str:
        return "PEER"


class PeerBlockPool:
    """Peer-resident KV blocks.  A block is one page of every KV tensor
    (layers, or K and V of each layer as vLLM's CanonicalKVCaches lists
    them); block b lives in slab b // slab_blocks, slot s = b % slab_blocks,
    and page t of it at slab_va + region[t] + s * page_sizes[t], where
    region[t] = slab_blocks * sum(page_sizes[:t]) (tensor-major, so a block's
    pages are equally spaced when the page sizes are equal).  Slabs are
    harvest_alloc'ed (Lossy) on first use; a revoked slab marks its blocks
    lost."""

    def __init__(self, runtime: HarvestRuntime, num_layers: int | None = None, page_bytes: int | None = None,
                 slab_blocks: int = 64, page_sizes=None):
        if page_sizes is None:
            if num_layers is None or page_bytes is None:
                raise ValueError("need page_sizes or num_layers and page_bytes")
            page_sizes = [page_bytes] * num_layers
        self.page_sizes = [int(x) for x in page_sizes]
        self.rt, self.slab_blocks = runtime, slab_blocks
        self.L, self.page = len(self.page_sizes), self.page_sizes[0]
        self.block_bytes = sum(self.page_sizes)
        self.region = np.concatenate([[0], np.cumsum(self.page_sizes)[:-1]]).astype(np.uint64) * np.uint64(slab_blocks)
        self.uniform = len(set(self.page_sizes)) == 1
        self.slabs: dict[int, object] = {}
        self.lost: set[int] = set()
        self.valid: set[int] = set()

    def _slab(self, idx: int):
        h = self.slabs.get(idx)
        if h is None or not self.rt.is_live(h):
            h = self.rt.harvest_alloc(self.slab_blocks * self.block_bytes,
                                      AllocationHints(durability=Durability.LOSSY, client_id="vllm-kv"))
            if h is None:
                return None
            self.rt.harvest_register_cb(h, lambda hh, reason, idx=idx: self._revoked(idx))
            self.slabs[idx] = h
        return h

    def _revoked(self, idx: int) -> None:
        lo = idx * self.slab_blocks
        for b in range(lo, lo + self.slab_blocks):
            if b in self.valid:
                self.valid.discard(b)
                self.lost.add(b)

    def is_resident(self, block_id: int) -> bool:
        """The block was stored and its slab has not been revoked since."""
        return int(block_id) in self.valid

    def release(self, block_id: int) -> None:
        """The manager dropped the block (evicted or lost): forget it."""
        self.valid.discard(int(block_id))
        self.lost.discard(int(block_id))

    def slot_bases(self, block_ids, for_store: bool) -> tuple[np.ndarray, list] | None:
        """slab_va + slot * page_sizes[0] per block (page 0's address when the
        page sizes are equal) and the slab handles touched."""
        bases = np.empty(len(block_ids), dtype=np.uint64)
        handles = {}
        for i, b in enumerate(block_ids):
            idx, slot = divmod(int(b), self.slab_blocks)
            h = self._slab(idx) if for_store else self.slabs.get(idx)
            if h is None or not self.rt.is_live(h):
                return None
            handles[idx] = h
            bases[i] = self.rt.address(h) + slot * self.page
        return bases, list(handles.values())

    def page_ptrs(self, block_ids, for_store: bool) -> tuple[np.ndarray, list] | None:
        """[L, n] page addresses of the given blocks."""
        r = self.slot_bases(block_ids, for_store)
        if r is None:
            return None
        bases, handles = r
        slots = (np.asarray(block_ids, dtype=np.uint64) % np.uint64(self.slab_blocks))
        slab0 = bases - slots * np.uint64(self.page)
        ps = np.asarray(self.page_sizes, dtype=np.uint64)[:, None]
        return slab0[None, :] + self.region[:, None] + slots[None, :] * ps, handles

    # layer stride of a block's pages (equal page sizes only)
    @property
    def layer_stride(self) -> int:
        return self.slab_blocks * self.page


class HarvestPeerHandler(OffloadingHandler):
    """OffloadingHandler for GPU <-> PEER KV transfers (one launch per job)."""

    def __init__(self, system, gpu_cache, pool: PeerBlockPool, engine: str = "auto", max_ctas: int = 0):
        """gpu_cache: a [num_layers, num_blocks, page_bytes] uint8 tensor
        (vLLM's per-layer KV tensors stacked), or a list of per-tensor
        [num_blocks, page_bytes] tensors (vLLM's CanonicalKVCaches.tensors,
        one page of each per block)."""
        self.sys, self.rt, self.pool = system, system.runtime, pool
        self.engine, self.max_ctas = N.ENGINES[engine], max_ctas
        self.stream = system.engine.stream
        self._jobs: dict[int, tuple] = {}
        self._done: list = []
        self.bind(gpu_cache)

    def bind(self, gpu_cache) -> None:
        """(Re)bind the GPU KV tensors the handler moves pages of.  A serving
        engine that re-initializes its KV cache (vLLM 0.22 can register the
        cache more than once) keeps this handler registered and rebinds it."""
        pool = self.pool
        if isinstance(gpu_cache, torch.Tensor):
            tensors = [gpu_cache[i] for i in range(gpu_cache.shape[0])]
        else:
            tensors = list(gpu_cache)
        if len(tensors) != pool.L:
            raise ValueError(f"{len(tensors)} KV tensors but the pool has {pool.L} pages per block")
        self.tensors = tensors
        self.nblocks = min(t.shape[0] for t in tensors)
        self.bases = np.array([t.data_ptr() for t in tensors], dtype=np.uint64)
        self.rows = np.array([t.stride(0) * t.element_size() for t in tensors], dtype=np.uint64)
        for t, ps in zip(tensors, pool.page_sizes):
            if t[0].numel() * t.element_size() < ps:
                raise ValueError("a KV tensor row is smaller than its page")
        self.L, self.page = pool.L, pool.page
        d = np.diff(self.bases.astype(np.int64))
        # whole-block form (K1 over the block table, 32 B of metadata per
        # block): equal pages, equally spaced tensors, rows of one page
        self.block_form = (pool.uniform and (len(d) == 0 or (d == d[0]).all() and d[0] > 0)
                           and (self.rows == np.uint64(pool.page)).all())
        self.layer_stride = int(d[0]) if len(d) else 0
        self.dev = tensors[0].device

    def _gpu_pages(self, block_ids) -> np.ndarray:
        b = np.asarray(block_ids, dtype=np.uint64)
        return self.bases[:, None] + b[None, :] * self.rows[:, None]

    def transfer_async(self, job_id: int, spec) -> bool:
        src, dst = spec
        if len(src.block_ids) != len(dst.block_ids):
            return False
        t0 = time.perf_counter()
        sm, dm = src.medium(), dst.medium()
        if sm == "GPU" and dm == "PEER":                                   # store (evict)
            gpu_ids, peer_ids = src.block_ids, dst.block_ids
            r = self.pool.page_ptrs(peer_ids, for_store=True)
            if r is None:
                return False
            for b in peer_ids:
                self.pool.valid.add(int(b))
                self.pool.lost.discard(int(b))
            kind = ("GPU", "PEER")
        elif sm == "PEER" and dm == "GPU":                                 # load (reload)
            gpu_ids, peer_ids = dst.block_ids, src.block_ids
            if any(not self.pool.is_resident(b) for b in peer_ids):
                _STATS["failed_loads"] += 1
                self._done.append(TransferResult(job_id, False, 0, 0.0, ("PEER", "GPU")))
                return True  # completes as failed: Lossy -> recompute
            r = self.pool.page_ptrs(peer_ids, for_store=False)
            if r is None:
                self._done.append(TransferResult(job_id, False, 0, 0.0, ("PEER", "GPU")))
                return True
            kind = ("PEER", "GPU")
        else:
            return False
        if len(gpu_ids) and int(np.max(gpu_ids)) >= self.nblocks:
            return False
        peer_pages, handles = r
        key = "store" if kind[0] == "GPU" else "load"
        _STATS[key + "_jobs"] += 1
        _STATS[key + "_blocks"] += len(gpu_ids)
        _STATS[key + "_bytes"] += len(gpu_ids) * self.pool.block_bytes
        gpu_pages = self._gpu_pages(gpu_ids)
        nb = len(gpu_ids)
        nbytes = nb * self.pool.block_bytes
        batch = self.rt.begin_reads(handles) if handles else None
        keep = ()
        if self.block_form:
            # one K1 launch over the block table: page (l, b) at base[b] + l*stride[b]
            gb, gs = gpu_pages[0], np.full(nb, self.layer_stride, dtype=np.uint64)
            pb, ps = peer_pages[0], np.full(nb, self.pool.layer_stride, dtype=np.uint64)
            sb, ss, db, ds = [np.ascontiguousarray(x, dtype=np.uint64)
                              for x in ((gb, gs, pb, ps) if kind[0] == "GPU" else (pb, ps, gb, gs))]
            N.call("hv_kv_gather_blocks_h", sb.ctypes.data, ss.ctypes.data, db.ctypes.data, ds.ctypes.data, nb,
                   self.L, self.page, self.sys.engine.engine, self.sys.engine.max_ctas, self.stream)
        else:
            # general layout: one launch over every page (per-page pointers and sizes)
            src_p, dst_p = (gpu_pages, peer_pages) if kind[0] == "GPU" else (peer_pages, gpu_pages)
            sizes = np.repeat(np.asarray(self.pool.page_sizes, dtype=np.uint64), nb)
            N.call("hv_swap_blocks_batch", np.ascontiguousarray(src_p.reshape(-1)).ctypes.data,
                   np.ascontiguousarray(dst_p.reshape(-1)).ctypes.data, sizes.ctypes.data, sizes.size,
                   self.sys.engine.engine, self.sys.engine.max_ctas, self.stream)

        def _finish(_x, keep=keep, batch=batch):
            if batch is not None:
                self.rt.end_reads(batch)
            self._done.append(TransferResult(job_id, True, nbytes, time.perf_counter() - t0, kind))

        self.sys.engine.track([_finish])
        self._jobs[job_id] = kind
        return True

    def get_finished(self) -> list:
        self.sys.loop.poll()
        out, self._done = self._done, []
        for r in out:
            self._jobs.pop(r.job_id, None)
        return out

    def wait(self, job_ids) -> None:
        while any(j in self._jobs for j in job_ids):
            self.sys.engine.wait_one()
            self.sys.loop.poll()
            done = {r.job_id for r in self._done}
            for j in list(job_ids):
                if j in done:
                    self._jobs.pop(j, None)

    def shutdown(self) -> None:
        self.sys.engine.synchronize()
        self.sys.loop.poll()
        if _WORKER_POOL[0] is self.pool:   # no later manager of this process reads a finished engine's pool
            _WORKER_POOL[0] = None


@dataclass
class _Entry:
    block_id: int
    ready: bool = False
    ref_cnt: int = 0


class HarvestOffloadingManager(OffloadingManager):
    """Scheduler-side manager of the PEER medium (vllm/v1/kv_offload/base.py:110-237).

    ``num_blocks`` peer block ids (the id space of the worker's
    PeerBlockPool) are handed out by prepare_store and recycled LRU-first.
    ``residency`` (an object with ``is_resident(block_id)`` and
    ``release(block_id)``, normally the worker's PeerBlockPool, or a callable
    returning it) is consulted on every lookup: a block whose slab was
    revoked since it was stored is a MISS -- the entry is dropped, its id
    freed and a removed event emitted -- so the scheduler recomputes it
    instead of loading bytes that are gone.  With no residency view (a
    scheduler process separate from the workers), revocations surface as
    failed loads (``TransferResult.success=False``) instead."""

    def __init__(self, num_blocks: int, residency=None, enable_events: bool = False):
        if num_blocks < 0:
            raise ValueError("num_blocks must be >= 0")
        self.medium = PeerBlocks.medium()
        self.num_blocks = num_blocks
        self._free = list(range(num_blocks - 1, -1, -1))
        self._entries: "OrderedDict[bytes, _Entry]" = OrderedDict()   # LRU order: oldest first
        self._residency = residency
        self.events: list | None = [] if enable_events else None
        self.stats = {"revoked_misses": 0, "evicted": 0}

    def _view(self):
        r = self._residency
        return r() if callable(r) and not hasattr(r, "is_resident") else r

    def _drop(self, key, e: _Entry, lost: bool) -> None:
        del self._entries[key]
        self._free.append(e.block_id)
        view = self._view()
        if view is not None:
            view.release(e.block_id)
        if lost:
            self.stats["revoked_misses"] += 1
        if self.events is not None:
            self.events.append(OffloadingEvent(keys=[key], medium=self.medium, removed=True))

    def lookup(self, key, req_context=None) -> bool | None:
        e = self._entries.get(key)
        if e is None:
            return False
        if not e.ready:
            return None                      # store in flight: retry later
        view = self._view()
        if view is not None and not view.is_resident(e.block_id):
            if e.ref_cnt == 0:
                self._drop(key, e, lost=True)
            return False                     # revoked: a miss, vLLM recomputes
        return True

    def prepare_load(self, keys, req_context=None) -> "PeerBlocks":
        ids = []
        for k in keys:
            e = self._entries.get(k)
            assert e is not None and e.ready, f"block {k!r} is not offloaded and ready"
            e.ref_cnt += 1
            ids.append(e.block_id)
        return PeerBlocks(ids)

    def touch(self, keys, req_context=None) -> None:
        for k in keys:
            if k in self._entries:
                self._entries.move_to_end(k)

    def complete_load(self, keys, req_context=None) -> None:
        for k in keys:
            e = self._entries.get(k)
            assert e is not None and e.ref_cnt > 0, f"block {k!r} was not being loaded"
            e.ref_cnt -= 1

    def prepare_store(self, keys, req_context=None) -> "PrepareStoreOutput | None":
        keys = list(keys)
        protected = set(keys)
        to_store = [k for k in keys if k not in self._entries]
        need = len(to_store) - len(self._free)
        evicted = []
        if need > 0:
            cands = [k for k, e in self._entries.items() if e.ready and e.ref_cnt == 0 and k not in protected]
            if len(cands) < need:
                return None
            for k in cands[:need]:
                self._drop(k, self._entries[k], lost=False)
                evicted.append(k)
            self.stats["evicted"] += len(evicted)
            if self.events is not None and evicted:   # _drop emitted one event per key: merge them
                del self.events[-len(evicted):]
                self.events.append(OffloadingEvent(keys=evicted, medium=self.medium, removed=True))
        ids = []
        for k in to_store:
            e = _Entry(self._free.pop())
            self._entries[k] = e
            ids.append(e.block_id)
        return PrepareStoreOutput(keys_to_store=to_store, store_spec=PeerBlocks(ids), evicted_keys=evicted)

    def complete_store(self, keys, req_context=None, success: bool = True) -> None:
        stored = []
        for k in keys:
            e = self._entries.get(k)
            if e is None or e.ready:
                continue
            if success:
                e.ready = True
                stored.append(k)
            else:
                del self._entries[k]
                self._free.append(e.block_id)
        if stored and self.events is not None:
            self.events.append(OffloadingEvent(keys=stored, medium=self.medium, removed=False))

    def take_events(self):
        if self.events:
            out, self.events = self.events, []
            yield from out

    def reset_cache(self) -> None:
        for k, e in list(self._entries.items()):
            if e.ref_cnt == 0:
                self._drop(k, e, lost=False)

    def shutdown(self) -> None:
        return


class HarvestOffloadingSpec(OffloadingSpec):
    """``kv_connector_extra_config = {"spec_name": "HarvestOffloadingSpec",
    "peer_bytes_to_use": <bytes of donor HBM to harvest>, "slab_blocks": 64,
    "donors": [<CUDA device ids>]}`` (donors default: every other visible
    GPU; a single-GPU box uses its own HBM as the stand-in donor).

    Worker side: a HarvestSystem on the worker's GPU with a VMM pool per
    donor, a PeerBlockPool laid out for the canonical KV tensors, and one
    HarvestPeerHandler serving both directions.  Scheduler side: a
    HarvestOffloadingManager over the same block id space; in one process
    it reads the pool's residency, so revocations become lookup misses."""

    def __init__(self, vllm_config, kv_cache_config):
        super().__init__(vllm_config, kv_cache_config)
        if getattr(self, "block_size_factor", 1) != 1:
            raise ValueError("HarvestOffloadingSpec moves whole GPU blocks (block_size_factor 1)")
        peer_bytes = int(self.extra_config.get("peer_bytes_to_use", 0))
        if peer_bytes <= 0:
            raise ValueError("peer_bytes_to_use must be given in kv_connector_extra_config")
        world = vllm_config.parallel_config.world_size
        if kv_cache_config.num_blocks > 0:
            total = sum(t.size for t in kv_cache_config.kv_cache_tensors)
            self.block_bytes = total // kv_cache_config.num_blocks
        else:
            self.block_bytes = 0
        self.peer_bytes = peer_bytes
        self.num_blocks = peer_bytes // (self.block_bytes * max(1, world)) if self.block_bytes else 0
        self.slab_blocks = int(self.extra_config.get("slab_blocks", 64))
        self.donors = self.extra_config.get("donors")
        self._manager = None
        self._pool = None
        self._handler = None
        self.system = None

    def get_manager(self):
        if self._manager is None:
            kec = getattr(self.vllm_config, "kv_events_config", None)
            events = bool(kec is not None and getattr(kec, "enable_kv_cache_events", False))
            # in-process engines (VLLM_ENABLE_V1_MULTIPROCESSING=0) build one
            # spec per role: the scheduler's manager sees the worker's pool
            self._manager = HarvestOffloadingManager(
                self.num_blocks, residency=lambda: self._pool if self._pool is not None else _WORKER_POOL[0],
                enable_events=events)
        return self._manager

    def _build_worker(self, tensors, page_sizes):
        from .system import HarvestSystem
        dev = tensors[0].device.index if tensors[0].device.index is not None else torch.cuda.current_device()
        donors = self.donors
        if donors is None:
            donors = [d for d in range(torch.cuda.device_count()) if d != dev] or [dev]
        block_bytes = sum(page_sizes)
        slabs = -(-self.num_blocks // self.slab_blocks)
        per_donor = -(-slabs // len(donors)) * self.slab_blocks * block_bytes
        self.system = HarvestSystem(dev, donors=list(donors), donor_bytes=max(per_donor, block_bytes * self.slab_blocks),
                                    host_bytes=1, local_bytes=1)
        self._pool = PeerBlockPool(self.system.runtime, slab_blocks=self.slab_blocks, page_sizes=page_sizes)
        _WORKER_POOL[0] = self._pool
        self._handler = HarvestPeerHandler(self.system, tensors, self._pool)

    def get_handlers(self, kv_caches):
        tensors = [t.tensor for t in kv_caches.tensors]
        page_sizes = [t.page_size_bytes for t in kv_caches.tensors]
        if self._handler is not None:
            # a second registration of the engine's KV cache (vLLM 0.22
            # re-initializes it): the worker already holds this handler for
            # both directions, so rebind it to the new tensors and register
            # nothing twice (the worker asserts on a repeated transfer type)
            if list(page_sizes) != list(self._pool.page_sizes):
                raise ValueError("re-registered KV cache with a different page layout")
            self._handler.bind(tensors)
            return
        self._build_worker(tensors, page_sizes)
        gpu_spec = _gpu_spec_type()
        yield gpu_spec, PeerBlocks, self._handler
        yield PeerBlocks, gpu_spec, self._handler


def _gpu_spec_type():
    if HAVE_VLLM:
        from vllm.v1.kv_offload.base import GPULoadStoreSpec  # type: ignore
        return GPULoadStoreSpec
    return GPUBlocks


_WORKER_POOL = [None]   # the peer pool the worker side of this process built (see get_manager)
_STATS = {"store_jobs": 0, "store_blocks": 0, "store_bytes": 0, "load_jobs": 0, "load_blocks": 0, "load_bytes": 0,
          "failed_loads": 0}


def handler_stats() -> dict:
    """Jobs, blocks and bytes every HarvestPeerHandler of this process has
    launched (stores GPU -> PEER, loads PEER -> GPU) and loads failed because
    a block was revoked."""
    return dict(_STATS)


def register_with_vllm() -> bool:
    """Make "HarvestOffloadingSpec" resolvable by OffloadingSpecFactory
    (vllm/v1/kv_offload/factory.py:21-32); idempotent."""
    if not HAVE_VLLM:
        return False
    from vllm.v1.kv_offload.factory import OffloadingSpecFactory  # type: ignore
    if "HarvestOffloadingSpec" not in OffloadingSpecFactory._registry:
        OffloadingSpecFactory.register_spec("HarvestOffloadingSpec", __name__, "HarvestOffloadingSpec")
    return True


register_with_vllm()
