"""vLLM KV-offload "peer" medium backed by harvested peer HBM.

PAPER.md §5.2 (lines 308-314) extends vLLM's KV manager with a
KVOffloadManager and a per-device OffloadingHandler.  vLLM 0.22's handler
contract is (vllm/v1/kv_offload/worker/worker.py:26-75):
    transfer_async(job_id, (src_spec, dst_spec)) -> bool
    get_finished() -> list[TransferResult]
    wait(job_ids) -> None
Its CPU handler moves blocks with swap_blocks_batch / cuMemcpyBatchAsync
(vllm/v1/kv_offload/cpu/gpu_worker.py:329).  ``HarvestPeerHandler`` implements
the same contract for GPU <-> PEER transfers.
- Destination/source pages are resolved from a ``PeerBlockPool`` (harvested
  slabs, one revocable handle per slab).
- Every job is ONE K1 launch over per-page pointers on the handler's stream.
- Loads that touch a block whose slab was revoked complete with success=False,
  i.e. Lossy semantics: vLLM recomputes.
vLLM is imported lazily; without it, minimal stand-ins of its spec/result
types are used so the adapter stays importable and testable.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .runtime import AllocationHints, Durability, HarvestRuntime

try:  # vLLM >= 0.22 layout
    from vllm.v1.kv_offload.worker.worker import OffloadingHandler, TransferResult  # type: ignore
    from vllm.v1.kv_offload.base import LoadStoreSpec  # type: ignore
    HAVE_VLLM = True
except Exception:  # pragma: no cover - exercised when vLLM is absent
    HAVE_VLLM = False

    class OffloadingHandler:  # minimal stand-in
        pass

    @dataclass
    class TransferResult:
        job_id: int
        success: bool
        transfer_size: int | None = None
        transfer_time: float | None = None
        transfer_type: tuple | None = None

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
    """Peer-resident KV blocks: block b lives in slab b // slab_blocks; layer l
    of slot s is at slab_va + (l * slab_blocks + s) * page_bytes.  Slabs are
    harvest_alloc'ed on first use; a revoked slab marks its blocks lost."""

    def __init__(self, runtime: HarvestRuntime, num_layers: int, page_bytes: int, slab_blocks: int = 64):
        self.rt, self.L, self.page, self.slab_blocks = runtime, num_layers, page_bytes, slab_blocks
        self.slabs: dict[int, object] = {}
        self.lost: set[int] = set()
        self.valid: set[int] = set()

    def _slab(self, idx: int):
        h = self.slabs.get(idx)
        if h is None or not self.rt.is_live(h):
            h = self.rt.harvest_alloc(self.slab_blocks * self.L * self.page,
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

    def page_bases(self, block_ids, for_store: bool) -> tuple[np.ndarray, np.ndarray, list] | None:
        """(base, layer_stride) per block and the slab handles touched."""
        bases = np.empty(len(block_ids), dtype=np.uint64)
        handles = {}
        for i, b in enumerate(block_ids):
            idx, slot = divmod(int(b), self.slab_blocks)
            h = self._slab(idx) if for_store else self.slabs.get(idx)
            if h is None or not self.rt.is_live(h):
                return None
            handles[idx] = h
            bases[i] = self.rt.address(h) + slot * self.page
        strides = np.full(len(block_ids), self.slab_blocks * self.page, dtype=np.uint64)  # [layer][slot]
        return bases, strides, list(handles.values())


class HarvestPeerHandler(OffloadingHandler):
    """OffloadingHandler for GPU <-> PEER KV transfers over K1."""

    def __init__(self, system, gpu_cache: torch.Tensor, pool: PeerBlockPool, engine: str = "auto",
                 max_ctas: int = 0):
        """gpu_cache: [num_layers, num_blocks, page_bytes] uint8 (layer-major,
        vLLM's per-layer KV tensors stacked)."""
        self.sys, self.rt, self.pool = system, system.runtime, pool
        self.cache = gpu_cache
        self.L, self.nblocks, self.page = gpu_cache.shape
        self.engine, self.max_ctas = N.ENGINES[engine], max_ctas
        self.dev = gpu_cache.device
        self.stream = system.engine.stream
        self._jobs: dict[int, tuple] = {}
        self._done: list = []

    def _gpu_bases(self, block_ids) -> tuple[np.ndarray, np.ndarray]:
        base = np.uint64(self.cache.data_ptr())
        b = base + np.asarray(block_ids, dtype=np.uint64) * np.uint64(self.page)
        return b, np.full(len(block_ids), self.nblocks * self.page, dtype=np.uint64)

    def transfer_async(self, job_id: int, spec) -> bool:
        src, dst = spec
        if len(src.block_ids) != len(dst.block_ids):
            return False
        t0 = time.perf_counter()
        if isinstance(src, GPUBlocks) and isinstance(dst, PeerBlocks):      # store (evict)
            sb, ss = self._gpu_bases(src.block_ids)
            r = self.pool.page_bases(dst.block_ids, for_store=True)
            if r is None:
                return False
            db, ds, handles = r
            for b in dst.block_ids:
                self.pool.valid.add(int(b))
                self.pool.lost.discard(int(b))
            kind = ("GPU", "PEER")
        elif isinstance(src, PeerBlocks) and isinstance(dst, GPUBlocks):    # load (reload)
            if any(int(b) not in self.pool.valid for b in src.block_ids):
                self._done.append(TransferResult(job_id, False, 0, 0.0, ("PEER", "GPU")))
                return True  # completes as failed: Lossy -> recompute
            r = self.pool.page_bases(src.block_ids, for_store=False)
            if r is None:
                self._done.append(TransferResult(job_id, False, 0, 0.0, ("PEER", "GPU")))
                return True
            sb, ss, handles = r
            db, ds = self._gpu_bases(dst.block_ids)
            kind = ("PEER", "GPU")
        else:
            return False
        # one K1 launch over the block table: page (l, b) at base[b] + l*stride[b]
        nb = len(sb)
        arrs = np.concatenate([np.broadcast_to(np.asarray(x, dtype=np.uint64), (nb,)) for x in (sb, ss, db, ds)])
        pinned = torch.from_numpy(arrs.view(np.int64)).pin_memory()
        with torch.cuda.stream(torch.cuda.ExternalStream(self.stream, device=self.dev)):   # the writer's pool
            dbuf = torch.empty(pinned.numel(), dtype=torch.int64, device=self.dev)
        N.call("hv_memcpy_h2d", dbuf.data_ptr(), pinned.data_ptr(), pinned.numel() * 8, self.stream)
        batch = self.rt.begin_reads(handles) if handles else None
        nbytes = nb * self.L * self.page

        def _finish(_x, keep=(pinned, dbuf), batch=batch):
            if batch is not None:
                self.rt.end_reads(batch)
            self._done.append(TransferResult(job_id, True, nbytes, time.perf_counter() - t0, kind))

        p = dbuf.data_ptr()
        N.call("hv_kv_gather_blocks", p, p + 8 * nb, p + 16 * nb, p + 24 * nb, nb, self.L, self.page,
               self.sys.engine.engine, self.sys.engine.max_ctas, self.stream)
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
