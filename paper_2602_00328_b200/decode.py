"""Pipelined MoE decode with expert weights served by Harvest tiers.

Reference semantics: moe._DecodeRun (moe.py:211-340).
- Stages (layer, micro-batch) run in layer-major order.
- The weights of stage s+1 are fetched while stage s computes ("issue fetches
  for stage s+1 at the start of stage s", moe.py:327-340).
- A stage starts when compute(s-1) is done AND every fetch of s has arrived.
Here the compute is real, not a constant per stage: a router GEMM, top-k, and
a SwiGLU expert FFN (bf16, cuBLAS batched GEMMs on the compute stream). The
fetch is the K2 kernel on the fetch stream, and "arrived" is a CUDA event.

B200-native choices:
- The fetch plan is built ON THE DEVICE. Router -> top-k -> active-expert
  mask -> per-expert size (0 when inactive), against a device copy of the
  residency address table, then one hv_batch_copy over all E descriptors.
  Zero-size descriptors are skipped by the kernel. No host synchronisation
  happens anywhere in a decode step, so the whole step can be captured in a
  CUDA graph.
- Two staging buffers alternate between stages. The compute of stage s reads
  buffer s%2 while the fetch of s+1 fills buffer (s+1)%2; a fetch waits for
  the compute that last read its buffer.
- Every expert slot of the staging buffer is zero-initialised, so inactive
  slots hold finite bytes. Their combine weight is exactly 0, which lets the
  FFN run densely over all E experts with fixed shapes.
- Drain: a stage may read any peer handle of its layer, so all of them join
  the stage's in-flight set (a superset of the reference's per-expert sets,
  which keeps drain-before-free).

fused=True consumes each expert where it lies instead (csrc/hv_ffn.cu): the
routed (token, expert) pairs are sorted by expert on the device and two
kernels stream the gate/up and down weight tiles straight from the resident
copy (donor HBM over NVLink, host over PCIe, local HBM) into mma.sync, then a
fixed-order top-k combine.  No staging buffer and no K2 launch; the bytes
cross the link once and the transfer overlaps the math tile by tile.  The
drain set of a fused step is every peer handle the step may read.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as TF

from . import _native as N
from ._nvtx import annotate
from .moe import ExpertFetcher


class MoEDecoder:
    # router / top-k / pair sort and the top-k combine + residual as library
    # kernels (hv_moe_route, hv_moe_combine); False: the torch ops (A/B)
    glue = True
    # the stage's library kernels (route, K4 gate/up, K4 down, combine) as a
    # chain of programmatic dependent launches: each one's prologue and launch
    # overlap the previous one's tail (needs the glue and 128-row tiles)
    pdl = True

    def __init__(self, fetcher: ExpertFetcher, tokens: int, microbatches: int = 1, seed: int = 0,
                 engine: str = "auto", max_ctas: int = 0, router_scale: float = 0.5,
                 residual_scale: float = 1.0, trace: bool = False, fused: bool = False,
                 host_plan: bool = False):
        m = fetcher.model
        if not (m.hidden and m.intermediate):
            raise ValueError("model profile needs hidden/intermediate sizes")
        if tokens % microbatches:
            raise ValueError("tokens must split evenly into micro-batches")
        self.f, self.m, self.rt = fetcher, m, fetcher.rt
        self.engine_id = N.ENGINES[engine]
        self.max_ctas = max_ctas
        eng = fetcher.engine
        self.dev = torch.device(f"cuda:{eng.cuda_device}")
        self.L, self.E, self.H, self.I, self.S = m.num_layers, m.num_experts, m.hidden, m.intermediate, m.expert_size
        self.T, self.nmb = tokens, microbatches
        # trace=True: timing events around every fetch (fetch stream) and every
        # expert FFN (compute stream) -> overlap_report()
        self.trace = trace
        self._tr: dict = {}
        # h <- h + residual_scale * moe(h); a power of two keeps it exact in bf16
        self.residual_scale = residual_scale
        self.tmb = tokens // microbatches
        g = torch.Generator().manual_seed(seed)
        self.router = [(torch.randn(self.E, self.H, generator=g) * router_scale / self.H ** 0.5)
                       .to(torch.bfloat16).to(self.dev) for _ in range(self.L)]
        self.x0 = (torch.randn(tokens, self.H, generator=g) * 0.5).to(torch.bfloat16).to(self.dev)
        # at most K experts can be active in one stage: K compact staging slots
        # per buffer; expert e goes to slot rank(e) among the active ones
        self.K = min(self.E, (tokens // microbatches) * m.top_k)
        self.fused = fused
        # host_plan=True (staged, eager): each stage's fetch plan is read back
        # to the host once its routing is done and handed to the library's
        # engine per source, so host-tier experts ride the copy engine
        # (55.5 GB/s over PCIe where the SM kernel reaches 51.4).  The host
        # waits for each stage's router -- the stage's fetch cannot start
        # before it anyway -- so this mode cannot be captured as a graph.
        self.host_plan = host_plan
        if host_plan and fused:
            raise ValueError("host_plan applies to the staged decoder")
        # experts stored as HV_FFN_TILED tiles (ExpertStore.fill_host(layout=
        # "tiled")): both decoders compute with K4, whose weight tiles then
        # arrive as one bulk copy each -- fused in place, staged over its
        # staging slots (the staged FFN's cuBLAS bmm reads row-major bytes)
        self.tiled = getattr(fetcher.store, "layout", "row") == "tiled"
        if fused or self.tiled:
            mt = N.c_int_out("hv_expert_ffn_max_tokens")
            if self.tmb > mt:
                raise ValueError(f"K4 decode: at most {mt} tokens per micro-batch")
            if self.I % 64 or self.H % 64:
                raise ValueError("K4 decode needs hidden and intermediate sizes that are multiples of 64")
        self.ffn_flags = N.FFN_TILED if self.tiled else 0
        # router logits scratch and the route kernel's arrival ticket (zeroed
        # here; the kernel re-arms it); the routed pairs of each staging slot
        # (the route kernel's limits: up to 256 experts, top-8, 256 tokens per stage)
        self.glue = type(self).glue and self.E <= 256 and m.top_k <= 8 and self.tmb <= 256 and self.H % 8 == 0
        self.pdl = type(self).pdl and self.glue and self.I % 128 == 0 and self.H % 128 == 0
        self._logits = torch.empty(self.tmb * self.E, dtype=torch.float32, device=self.dev)
        self._ticket = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._pairs = [None, None]
        # fused mode reads peer / local experts in place; only host-tier
        # experts are staged (one buffer: K2 and K4 run in order on one stream)
        self.staging = [torch.zeros(self.K, self.S, dtype=torch.uint8, device=self.dev)
                        for _ in range(1 if fused else 2)]
        self.slot_base = [b.data_ptr() for b in self.staging]
        self.dst_ptrs = [torch.zeros(self.E, dtype=torch.int64, device=self.dev) for _ in range(2)]
        self.idx_ext = [torch.zeros(self.K + 1, dtype=torch.int64, device=self.dev) for _ in range(2)]
        self.idx = [x[:self.K] for x in self.idx_ext]
        self._earange = torch.arange(self.E, device=self.dev)
        self.valid = [torch.zeros(self.K, dtype=torch.bool, device=self.dev) for _ in range(2)]
        self._kslots = torch.arange(self.K, device=self.dev)
        self.compute = torch.cuda.Stream(self.dev)
        self.fetch_stream_h = eng.stream
        self.fetch = torch.cuda.ExternalStream(eng.stream, device=self.dev)
        self.sync_tables()
        n = self.L * self.nmb
        self.sizes = [torch.zeros(self.E, dtype=torch.int64, device=self.dev) for _ in range(2)]
        self.comb = [torch.zeros(self.tmb, self.E, dtype=torch.float32, device=self.dev) for _ in range(2)]
        self.stages = [(layer, mb) for layer in range(self.L) for mb in range(self.nmb)]
        self.bytes_fetched_per_step = None
        self._n_stages = n

    # ---------------------------------------------------------------- tables
    def _table_host(self) -> tuple[torch.Tensor, torch.Tensor]:
        # LOCAL experts are staged from their resident copy in HBM (a device-
        # local copy); PEER/HOST experts are the fetches the reference counts
        src = np.where(self.f.tier == 0, self.f.local_addr, self.f.src_addr).astype(np.uint64)
        if np.any(src == 0):
            raise ValueError("an expert has no source address (LOCAL tier needs ExpertFetcher(local_addr=...))")
        if self.fused and np.any(src % 16):
            raise ValueError("fused decode reads experts with 16-byte cp.async: expert objects must be 16-byte aligned")
        self._addr_host = src.copy()
        return torch.from_numpy(src.view(np.int64).copy()), torch.from_numpy((self.f.tier != 0).copy())

    def sync_tables(self) -> None:
        """Upload the residency address table and fetch mask (call after
        placement or revocation changed ExpertFetcher's tables)."""
        if getattr(self, "_graph", None) is not None:
            return self._sync_tables_in_place()
        new_addr, new_fetchable = self._table_host()
        if getattr(self, "addr", None) is None:
            # two device copies of the table: in-flight fetch kernels read the
            # current one through raw pointers while the next one is written
            self._addr_bufs = [new_addr.to(self.dev), new_addr.to(self.dev)]
            self._addr_done = [None, None]
            self._addr_cur = 0
            self.addr = self._addr_bufs[0]
            self.fetchable = new_fetchable.to(self.dev)
            self.hosttier = torch.from_numpy(self.f.tier == 2).to(self.dev)
        else:
            nxt = 1 - self._addr_cur
            if self._addr_done[nxt] is not None:
                self._addr_done[nxt].synchronize()   # last step that read buffer nxt is done
            self._addr_bufs[nxt].copy_(new_addr)
            self.fetchable.copy_(new_fetchable)
            self.hosttier.copy_(torch.from_numpy(self.f.tier == 2))
            self._addr_cur = nxt
            self.addr = self._addr_bufs[nxt]
        self.layer_handles = [[h for (l, _e), h in self.f.handles.items() if l == layer] for layer in range(self.L)]
        self._any_host = (self.f.tier == 2).any(axis=1).tolist()
        self._table_version = getattr(self.f, "version", 0)

    def _sync_tables_in_place(self) -> None:
        """Graph mode: the captured kernels read one fixed table, so the new
        table is copied into it on the replay stream, ordered after every
        earlier replay and before the next (no host synchronisation)."""
        new_addr, new_fetchable = self._table_host()
        cur = torch.cuda.current_stream(self.dev)
        pinned = new_addr.pin_memory()
        with torch.cuda.stream(cur):
            self.addr.copy_(pinned, non_blocking=True)
            self.fetchable.copy_(new_fetchable.pin_memory(), non_blocking=True)
            self.hosttier.copy_(torch.from_numpy(self.f.tier == 2).pin_memory(), non_blocking=True)
        self._staged_tables = (pinned, cur.record_event())   # keep the source alive until copied
        self.layer_handles = [[h for (l, _e), h in self.f.handles.items() if l == layer] for layer in range(self.L)]
        self._any_host = (self.f.tier == 2).any(axis=1).tolist()
        self._table_version = getattr(self.f, "version", 0)

    # ---------------------------------------------------------------- pieces
    def _route(self, h: torch.Tensor, layer: int, slot: int) -> None:
        comb = self.comb[slot]
        comb.zero_()
        if self.glue:
            probs, topi, counts, offs, tok, pos = self._route_k(h, layer)
            self._pairs[slot] = (probs, counts, offs, tok, pos)   # K4 over tiled staging slots reuses them
            comb.scatter_(1, topi, probs)
            active = counts > 0
        else:
            logits = (h @ self.router[layer].t()).float()
            topv, topi = logits.topk(self.m.top_k, dim=1)
            if self._counts is not None:
                self._counts[layer].index_add_(0, topi.reshape(-1), torch.ones_like(topi.reshape(-1)))
            probs = torch.softmax(topv, dim=1)
            comb.scatter_(1, topi, probs)
            active = (comb > 0).any(dim=0)
            self._pairs[slot] = None
        torch.where(active, torch.full_like(self.sizes[slot], self.S), torch.zeros_like(self.sizes[slot]),
                    out=self.sizes[slot])
        # compact placement: rank among active experts -> staging slot; the
        # K slot owners in order (active first, stable) for the FFN
        rank = torch.cumsum(active.to(torch.int64), 0) - 1
        # slot owners: scatter e into position rank(e) (inactive -> dummy slot K)
        ext = self.idx_ext[slot]
        ext.zero_()
        ext.scatter_(0, torch.where(active, rank, self.K), self._earange)
        torch.add(rank.clamp_(min=0) * self.S, self.slot_base[slot], out=self.dst_ptrs[slot])
        torch.lt(self._kslots, active.sum(), out=self.valid[slot])

    def _ffn(self, h: torch.Tensor, slot: int, buf: int, layer: int) -> torch.Tensor:
        """The stage's expert FFN over the staging slots; returns the new h
        (h + residual_scale * moe(h))."""
        if self.tiled:
            # K4 over the staging slots: dst_ptrs[slot][e] is active expert e's
            # slot; the routed pairs are _route's (or recomputed on the same inputs)
            pr = self._pairs[slot] if self._pairs[slot] is not None else self._route_pairs(h, layer, count=False)
            return self._k4(h, self.dst_ptrs[slot], *pr, torch.cuda.current_stream(self.dev).cuda_stream)
        K, I, H = self.K, self.I, self.H
        w = self.staging[buf].view(torch.bfloat16).view(K, 3 * I * H)
        gate = w[:, :I * H].view(K, I, H)
        up = w[:, I * H:2 * I * H].view(K, I, H)
        down = w[:, 2 * I * H:].view(K, H, I)
        x = h.unsqueeze(0).expand(K, h.shape[0], H)
        a = TF.silu(torch.bmm(x, gate.transpose(1, 2))) * torch.bmm(x, up.transpose(1, 2))
        y = torch.bmm(a, down.transpose(1, 2))                       # [K, T, H]
        # combine weights of the slot owners; unused slots (stale but finite
        # bytes) get weight exactly 0
        wk = self.comb[slot].index_select(1, self.idx[slot]) * self.valid[slot].to(torch.float32)
        wts = wk.t().unsqueeze(-1).to(y.dtype)                       # [K, T, 1]
        return self._residual(h, (y * wts).sum(0))

    def _residual(self, h: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        return h + (y * self.residual_scale if self.residual_scale != 1.0 else y)

    def _issue_fetch(self, s: int, ready: torch.cuda.Event, buf_free: torch.cuda.Event | None) -> torch.cuda.Event:
        layer, _ = self.stages[s]
        slot = s % 2
        self.fetch.wait_event(ready)
        if buf_free is not None:
            self.fetch.wait_event(buf_free)
        if self.trace:
            fs = torch.cuda.Event(enable_timing=True)
            fs.record(self.fetch)
        if self.host_plan and not self._capturing:
            ready.synchronize()                       # this stage's routing (its fetch plan) is done
            sizes = self.sizes[slot].cpu().numpy().view(np.uint64)
            act = np.nonzero(sizes)[0]
            src = np.ascontiguousarray(self._addr_host[layer, act])
            dst = np.ascontiguousarray(self.dst_ptrs[slot].cpu().numpy().view(np.uint64)[act])
            sz = np.ascontiguousarray(sizes[act])
            N.call("hv_swap_blocks_batch", src.ctypes.data, dst.ctypes.data, sz.ctypes.data, len(act),
                   N.ENGINE_AUTO, self.max_ctas, self.fetch_stream_h)
        else:
            N.call("hv_batch_copy", self.addr[layer].data_ptr(), self.dst_ptrs[slot].data_ptr(),
                   self.sizes[slot].data_ptr(), self.E, self.engine_id, self.max_ctas, self.fetch_stream_h)
        if self.trace:
            fe = torch.cuda.Event(enable_timing=True)
            fe.record(self.fetch)
            self._tr.setdefault(s, {})["fetch"] = (fs, fe)
        handles = self.layer_handles[layer]
        if handles and not self._capturing:   # graph mode: tracked per replay instead
            batch = self.rt.begin_reads(handles)
            self.f.engine.track([lambda _x, b=batch: self.rt.end_reads(b)])
        ev = torch.cuda.Event()
        ev.record(self.fetch)
        return ev

    # ---------------------------------------------------------------- step
    _capturing = False
    _graph = None
    _graph_exec = None
    _counts = None

    def __del__(self):
        try:
            if self._graph_exec is not None:
                N.lib().hv_graph_exec_destroy(self._graph_exec)
        except Exception:
            pass

    def routing_counts(self, x: torch.Tensor | None = None) -> np.ndarray:
        """Expert activation counts [L, E] of one eager step from ``x`` (the
        decoder's input by default): the ``RoutingTrace.counts`` that
        ``place_offloaded`` ranks experts by (moe.py:354-383)."""
        self._counts = torch.zeros(self.L, self.E, dtype=torch.int64, device=self.dev)
        try:
            x = self.x0 if x is None else x
            self._step_fused(x) if self.fused else self._step_eager(x)
            return self._counts.cpu().numpy()
        finally:
            self._counts = None

    @annotate("harvest.decode_step")
    def step(self, x: torch.Tensor) -> torch.Tensor:
        """One decode step over all layers; returns the new hidden states.
        Residency changes (revocation callbacks, re-placement arrivals) seen
        since the last step are uploaded first; within a step the table is a
        snapshot, and reads of a handle revoked meanwhile extend its drain.
        After capture_graph() the step is one CUDA graph replay."""
        self._settle_releases()
        if getattr(self.f, "version", 0) != self._table_version:
            self.sync_tables()
        if self._graph is not None:
            return self._replay(x)
        if self.fused:
            return self._step_fused(x)
        return self._step_eager(x)

    def _settle_releases(self) -> None:
        """A revoke/free that began on a handle this decoder reads is drained
        before the next step: wait for the reads already enqueued, let the
        runtime finish the release (invalidate -> callback -> free; the
        callback moves residency to the host copy), so the next step's table
        no longer names the handle.  Without this, steps enqueued back to back
        keep the handle's in-flight set non-empty and the drain never ends."""
        ep = self.rt.release_epoch
        if ep == getattr(self, "_release_seen", 0):
            return
        self._release_seen = ep
        if any(self.rt.is_draining(h) for hs in self.layer_handles for h in hs):
            torch.cuda.synchronize(self.dev)
            self.rt.sim.poll() if hasattr(self.rt.sim, "poll") else self.rt.sim.run()

    def capture_graph(self, node_priority: bool = False) -> None:
        """Capture one decode step (every stage's router, top-k, fetch plan,
        K2 fetch and expert FFN, on both streams) as a CUDA graph; later
        step() calls replay it.  Inputs are copied into a static buffer; the
        output tensor returned by step() is reused by the next replay.
        ``node_priority``: instantiate through the library with
        HV_GRAPH_NODE_PRIORITY, so kernel nodes captured from the fetch stream
        keep that stream's priority inside the replay."""
        if self.trace:
            raise ValueError("trace mode records per-launch events; capture without trace")
        if self.host_plan:
            raise ValueError("host_plan reads each stage's plan back to the host: it cannot be captured")
        if self._graph is not None:
            return
        self._graph_in = self.x0.clone()
        cur = torch.cuda.current_stream(self.dev)
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(cur)
        self._capturing = True
        try:
            body = self._step_fused if self.fused else self._step_eager
            with torch.cuda.stream(side):            # warm-up outside capture (allocator, cuBLAS handles)
                for _ in range(2):
                    body(self._graph_in)
            cur.wait_stream(side)
            torch.cuda.synchronize(self.dev)
            g = torch.cuda.CUDAGraph(keep_graph=node_priority)
            with torch.cuda.graph(g):
                self._graph_out = body(self._graph_in)
        finally:
            self._capturing = False
        torch.cuda.synchronize(self.dev)
        self._graph = g
        self._graph_exec = None
        if node_priority:
            ex = C.c_void_p()
            N.call("hv_graph_instantiate", C.c_void_p(g.raw_cuda_graph()), N.GRAPH_NODE_PRIORITY, C.byref(ex))
            self._graph_exec = ex

    def _replay(self, x: torch.Tensor) -> torch.Tensor:
        cur = torch.cuda.current_stream(self.dev)
        if x.data_ptr() != self._graph_in.data_ptr():
            self._graph_in.copy_(x)
        # drain bookkeeping for every peer handle the step may read
        handles = [h for hs in self.layer_handles for h in hs]
        batch = self.rt.begin_reads(handles) if handles else None
        if self._graph_exec is not None:
            N.call("hv_graph_launch", self._graph_exec, C.c_void_p(cur.cuda_stream))
        else:
            self._graph.replay()
        done = torch.cuda.Event()
        done.record(cur)
        self._addr_done[self._addr_cur] = done
        if batch is not None:
            self.fetch.wait_stream(cur)              # the tracking event fires after the replay
            self.f.engine.track([lambda _x, b=batch: self.rt.end_reads(b)])
        return self._graph_out

    def _step_eager(self, x: torch.Tensor) -> torch.Tensor:
        hs = list(x.view(self.nmb, self.tmb, self.H).clone().unbind(0))
        cur = torch.cuda.current_stream(self.dev)
        self.compute.wait_stream(cur)
        n = self._n_stages
        fetched = [None] * n
        buf_free = [None, None]
        with torch.cuda.stream(self.compute):
            layer0, mb0 = self.stages[0]
            self._route(hs[mb0], layer0, 0)
            ev = torch.cuda.Event()
            ev.record(self.compute)
        fetched[0] = self._issue_fetch(0, ev, None)
        for s in range(n):
            layer, mb = self.stages[s]
            slot = buf = s % 2
            with torch.cuda.stream(self.compute):
                nxt_ready = None
                if s + 1 < n and self.nmb > 1:   # stage s+1's input already exists
                    l2, mb2 = self.stages[s + 1]
                    self._route(hs[mb2], l2, (s + 1) % 2)
                    nxt_ready = torch.cuda.Event()
                    nxt_ready.record(self.compute)
                self.compute.wait_event(fetched[s])
                if self.trace:
                    cs = torch.cuda.Event(enable_timing=True)
                    cs.record(self.compute)
                hs[mb] = self._ffn(hs[mb], slot, buf, layer)
                if self.trace:
                    ce = torch.cuda.Event(enable_timing=True)
                    ce.record(self.compute)
                    self._tr.setdefault(s, {})["compute"] = (cs, ce)
                done = torch.cuda.Event()
                done.record(self.compute)
                buf_free[buf] = done
                if s + 1 < n and self.nmb == 1:  # next stage depends on this one
                    l2, mb2 = self.stages[s + 1]
                    self._route(hs[mb2], l2, (s + 1) % 2)
                    nxt_ready = torch.cuda.Event()
                    nxt_ready.record(self.compute)
            if s + 1 < n:
                fetched[s + 1] = self._issue_fetch(s + 1, nxt_ready, buf_free[(s + 1) % 2] if s >= 1 else None)
        cur.wait_stream(self.compute)
        done = torch.cuda.Event()
        done.record(cur)              # every fetch of this step read self.addr before this point
        self._addr_done[self._addr_cur] = done
        return torch.stack(hs).view(self.T, self.H)

    # ---------------------------------------------------------------- fused
    def _route_k(self, h: torch.Tensor, layer: int):
        """hv_moe_route: router logits (fp32), top-k, softmax and the routed
        pairs sorted by expert in one launch."""
        if not h.is_contiguous():
            h = h.contiguous()
        T, k, E = h.shape[0], self.m.top_k, self.E
        probs = torch.empty(T, k, dtype=torch.float32, device=self.dev)
        topi = torch.empty(T, k, dtype=torch.int64, device=self.dev)
        counts = torch.empty(E, dtype=torch.int32, device=self.dev)
        offs = torch.empty(E, dtype=torch.int32, device=self.dev)
        tok = torch.empty(T * k, dtype=torch.int32, device=self.dev)
        pos = torch.empty(T * k, dtype=torch.int64, device=self.dev)
        N.call("hv_moe_route", h.data_ptr(), self.router[layer].data_ptr(), T, self.H, E, k,
               self._logits.data_ptr(), probs.data_ptr(), topi.data_ptr(), counts.data_ptr(), offs.data_ptr(),
               tok.data_ptr(), pos.data_ptr(), self._ticket.data_ptr(), N.MOE_OVERLAP_PREVIOUS if self.pdl else 0,
               torch.cuda.current_stream(self.dev).cuda_stream)
        if self._counts is not None:
            self._counts[layer].index_add_(0, topi.reshape(-1), torch.ones_like(topi.reshape(-1)))
        return probs, topi, counts, offs, tok, pos

    def _route_k_nocount(self, h: torch.Tensor, layer: int):
        saved, self._counts = self._counts, None
        try:
            return self._route_k(h, layer)
        finally:
            self._counts = saved

    def _route_pairs(self, h: torch.Tensor, layer: int, count: bool = True):
        """Router -> top-k -> routed pairs sorted by expert, all on the device:
        counts/offsets per expert, the token row of each sorted pair, and the
        sorted position of pair (t, j) for the combine."""
        if self.glue:
            probs, _topi, counts, offs, tok, pos = self._route_k(h, layer) if count else self._route_k_nocount(h, layer)
            return probs, counts, offs, tok, pos
        k = self.m.top_k
        logits = (h @ self.router[layer].t()).float()
        topv, topi = logits.topk(k, dim=1)
        if count and self._counts is not None:
            self._counts[layer].index_add_(0, topi.reshape(-1), torch.ones_like(topi.reshape(-1)))
        probs = torch.softmax(topv, dim=1)
        flat = topi.reshape(-1)
        order = torch.argsort(flat, stable=True)
        counts = torch.zeros(self.E, dtype=torch.int32, device=self.dev)
        counts.scatter_add_(0, flat, torch.ones_like(flat, dtype=torch.int32))
        offs = (torch.cumsum(counts, 0, dtype=torch.int32) - counts)
        tok = torch.div(order, k, rounding_mode="floor").to(torch.int32)
        pos = torch.empty_like(order)
        pos[order] = torch.arange(order.numel(), device=self.dev)
        return probs, counts, offs, tok, pos

    def _ffn_fused(self, h: torch.Tensor, layer: int) -> torch.Tensor:
        probs, counts, offs, tok, pos = self._route_pairs(h, layer)
        stream = torch.cuda.current_stream(self.dev).cuda_stream
        addr = self.addr[layer]
        if self._capturing or self._any_host[layer]:
            # host-tier experts: K2 over PCIe into compact local slots first
            # (sequential reads, the PCIe-efficient path), then K4 reads those
            # slots and every peer / local expert in place
            if self.glue:
                dst = torch.empty(self.E, dtype=torch.int64, device=self.dev)
                sizes = torch.empty_like(dst)
                staged = torch.empty_like(dst)
                N.call("hv_moe_stage_plan", counts.data_ptr(), addr.data_ptr(), self.hosttier[layer].data_ptr(),
                       self.slot_base[0], self.S, self.E, dst.data_ptr(), sizes.data_ptr(), staged.data_ptr(), stream)
            else:
                stage = (counts > 0) & self.hosttier[layer]
                rank = torch.cumsum(stage.to(torch.int64), 0) - 1
                dst = torch.where(stage, rank * self.S + self.slot_base[0], 0)
                sizes = torch.where(stage, self.S, 0)
                staged = torch.where(stage, dst, addr)
            N.call("hv_batch_copy", addr.data_ptr(), dst.data_ptr(), sizes.data_ptr(), self.E, self.engine_id,
                   self.max_ctas, stream)
            addr = staged
        return self._k4(h, addr, probs, counts, offs, tok, pos, stream)

    def _k4(self, h, addr, probs, counts, offs, tok, pos, stream) -> torch.Tensor:
        """K4 (gate/up, then down) over the experts at `addr` and the top-k
        combine."""
        P, H, I = pos.numel(), self.H, self.I
        act = torch.empty(P, I, dtype=torch.bfloat16, device=self.dev)
        y = torch.empty(P, H, dtype=torch.float32, device=self.dev)
        w = addr.data_ptr()
        pdl_up = N.FFN_WAIT_PREVIOUS if self.pdl else 0
        N.call("hv_expert_ffn_gate_up_ex", w, counts.data_ptr(), offs.data_ptr(), tok.data_ptr(), h.data_ptr(),
               act.data_ptr(), self.E, H, I, self.ffn_flags | pdl_up, stream)
        # down as a programmatic dependent of gate/up: its first weight tiles
        # stream while gate/up drains (the mma.sync form measured slower this
        # way, r3b: 201.5 vs 195.4 us per Qwen stage; the tcgen05 form: §3)
        pdl_down = N.FFN_OVERLAP_PREVIOUS if self.pdl else 0
        N.call("hv_expert_ffn_down_ex", w, counts.data_ptr(), offs.data_ptr(), act.data_ptr(), y.data_ptr(), self.E,
               H, I, self.ffn_flags | pdl_down, stream)
        # top-k combine in a fixed order (deterministic, no atomics), plus the residual
        if self.glue:
            if not h.is_contiguous():
                h = h.contiguous()
            N.call("hv_moe_combine", y.data_ptr(), probs.data_ptr(), pos.data_ptr(), h.data_ptr(), h.shape[0], H,
                   self.m.top_k, float(self.residual_scale), N.MOE_OVERLAP_PREVIOUS if self.pdl else 0, stream)
            return h
        yt = y.index_select(0, pos).view(h.shape[0], self.m.top_k, H)
        return self._residual(h, (yt * probs.unsqueeze(-1)).sum(1).to(h.dtype))

    def _step_fused(self, x: torch.Tensor) -> torch.Tensor:
        hs = list(x.view(self.nmb, self.tmb, self.H).clone().unbind(0))
        cur = torch.cuda.current_stream(self.dev)
        self.compute.wait_stream(cur)
        handles = [hh for hl in self.layer_handles for hh in hl]
        batch = self.rt.begin_reads(handles) if (handles and not self._capturing) else None
        with torch.cuda.stream(self.compute):
            for s, (layer, mb) in enumerate(self.stages):
                if self.trace:
                    cs = torch.cuda.Event(enable_timing=True)
                    cs.record(self.compute)
                hs[mb] = self._ffn_fused(hs[mb], layer)
                if self.trace:
                    ce = torch.cuda.Event(enable_timing=True)
                    ce.record(self.compute)
                    self._tr.setdefault(s, {})["fused"] = (cs, ce)
        cur.wait_stream(self.compute)
        done = torch.cuda.Event()
        done.record(cur)
        self._addr_done[self._addr_cur] = done
        if batch is not None:               # the drain completes when the step's reads have
            self.fetch.wait_stream(cur)
            self.f.engine.track([lambda _x, b=batch: self.rt.end_reads(b)])
        return torch.stack(hs).view(self.T, self.H)

    def overlap_report(self) -> dict:
        """From the last traced step: per-stage fetch and FFN intervals on the
        device clock, and how much of each stage-(s+1) fetch ran while stage s
        computed (the CGOPipe overlap, moe.py:327-340)."""
        torch.cuda.synchronize(self.dev)
        stages = sorted(k for k, v in self._tr.items() if "fetch" in v and "compute" in v)
        if not stages:
            return {}
        base = self._tr[stages[0]]["fetch"][0]
        iv = {s: {k: (base.elapsed_time(a), base.elapsed_time(b)) for k, (a, b) in self._tr[s].items()}
              for s in stages}
        fetch_ms = sum(v["fetch"][1] - v["fetch"][0] for v in iv.values())
        comp_ms = sum(v["compute"][1] - v["compute"][0] for v in iv.values())
        ov = 0.0
        for s in stages:
            if s + 1 in iv:
                (f0, f1), (c0, c1) = iv[s + 1]["fetch"], iv[s]["compute"]
                ov += max(0.0, min(f1, c1) - max(f0, c0))
        span = max(v["compute"][1] for v in iv.values()) - min(v["fetch"][0] for v in iv.values())
        return {"stages": len(stages), "fetch_ms": fetch_ms, "compute_ms": comp_ms, "overlap_ms": ov,
                "compute_hidden_fraction": ov / comp_ms if comp_ms else None, "span_ms": span,
                "serial_ms": fetch_ms + comp_ms}

    def decode(self, steps: int, x: torch.Tensor | None = None) -> torch.Tensor:
        h = self.x0 if x is None else x
        for _ in range(steps):
            h = self.step(h)
            self.rt.sim.poll() if hasattr(self.rt.sim, "poll") else None
        return h


# ------------------------------------------------------------------ sweep
@dataclass(frozen=True)
class SweepRow:
    """moe.py:386-391.  ``stall_s``: fetch time the FFN did not hide, from a
    traced step's device clock (staged mode; None for fused, which has no
    separate fetch)."""
    fraction_pct: float
    tier: str
    tokens_per_s: float
    stall_s: float | None


def offload_sweep(system, model, fractions, tier, tokens: int = 32, microbatches: int = 2, seed: int = 0,
                  fused: bool = False, graph: bool = True, steps: int = 5, warmup: int = 2,
                  content_seed: int = 0) -> list[SweepRow]:
    """moe.offload_sweep (moe.py:394-415) on real decode: for each offload
    fraction, the coldest experts of every layer (ranked by the routing
    counts of one all-local step) go to ``tier`` -- PEER_HBM through
    ``place_offloaded``'s rebalance onto ``system``'s donor pools, HOST_DRAM
    read from the pinned host tier -- the rest stay LOCAL in a resident HBM
    copy, and a ``MoEDecoder`` is timed on the device clock.  Every
    fraction's output must equal the all-local output bit for bit (raises
    otherwise).  Peer handles are freed between fractions."""
    from .memalloc import Tier
    from .moe import ExpertResidency, ExpertStore, RoutingTrace, place_offloaded
    from .runtime import StaleHandleError
    if tier not in (Tier.PEER_HBM, Tier.HOST_DRAM):
        raise ValueError(f"offload tier must be peer or host, got {tier}")
    L, E, S = model.num_layers, model.num_experts, model.expert_size
    rt, loop = system.runtime, system.loop
    store = ExpertStore(model, system.host_id, system.host)
    store.fill_host(system.compute, weights=True)
    dev = torch.device(f"cuda:{system.compute}")
    resident = torch.from_numpy(system.host.view()[:L * E * S].copy()).to(dev)
    local_addr = [[resident.data_ptr() + (layer * E + e) * S for e in range(E)] for layer in range(L)]

    def decoder(residency):
        f = ExpertFetcher(rt, model, residency, store, local_addr=local_addr)
        return MoEDecoder(f, tokens=tokens, microbatches=microbatches, seed=seed, fused=fused)

    local = ExpertResidency(model)
    for layer in range(L):
        for e in range(E):
            local.set_tier(layer, e, Tier.LOCAL_HBM)
    d0 = decoder(local)
    counts = d0.routing_counts()
    want = d0.step(d0.x0).clone()
    trace = RoutingTrace(1, L, E, [], counts)
    rows = []
    for fraction in fractions:
        residency = ExpertResidency(model)
        place_offloaded(loop, rt, model, residency, trace, fraction, tier, system.host_id, store=store)
        dec = decoder(residency)
        got = dec.step(dec.x0)
        if not torch.equal(got, want):
            raise RuntimeError(f"offload_sweep: output at {fraction}% differs from the all-local decode")
        stall = None
        if not fused:
            tr = MoEDecoder(dec.f, tokens=tokens, microbatches=microbatches, seed=seed, trace=True)
            tr.step(tr.x0)
            rep = tr.overlap_report()
            stall = max(0.0, rep["span_ms"] - rep["compute_ms"]) * 1e-3 if rep else None
            del tr
        if graph:
            dec.capture_graph()
        for _ in range(warmup):
            dec.step(dec.x0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record()
        for _ in range(steps):
            dec.step(dec.x0)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
        rows.append(SweepRow(fraction, "peer" if tier == Tier.PEER_HBM else "host", tokens / (ms * 1e-3), stall))
        del dec
        torch.cuda.synchronize(dev)
        loop.run()
        for ent in residency.entries.values():
            if ent.handle is not None:
                try:
                    rt.harvest_free(ent.handle)
                except StaleHandleError:
                    pass
        loop.run()
    return rows
