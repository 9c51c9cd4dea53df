"""Decode attention over a paged KV cache whose blocks live in any Harvest tier.

The reference's KV module stops at moving blocks: reload
brings them back to local HBM, and the paper's KV experiment (Fig 7,
SPEC.md:426-434) reports the reload latency alone.  This is the consumer that
turns K1 into decode tokens/s: for every layer, K1 gathers that layer's page
of every block of every sequence -- from local HBM, a donor's slab over
NVLink, or the pinned host tier -- into a contiguous double buffer on the
fetch stream, and grouped-query attention for that layer runs on the compute
stream while the next layer's gather is in flight.

Unlike the MoE stage (routing of layer l+1 needs layer l's output), the KV
pages of every layer are known before the step starts, so the gathers run
ahead of the attention, bounded only by the two buffers: the step takes
max(sum of gathers, sum of attention) plus one stage.

Per step the block table is resolved once on the host
(KVCacheManager.page_table) and uploaded once; the per-layer source arrays
are one device-side broadcast, so each layer costs one K1 launch and no host
work.  The peer slabs read by the step form its drain set (begin_reads
before, the step's CUDA event after), so a revocation mid-step waits for the
gathers that read the slab.

The attention is hv_paged_decode_attention (csrc/hv_attn.cu), a split-K
flash-decoding kernel over a table of page pointers.  fused=True skips K1:
the attention reads every page where it lies (peer slab over NVLink, host
over PCIe, local HBM), so each KV byte crosses the link once and is never
written locally.  Both modes run the same kernel on the same bytes, so their
outputs are bit-identical.

Page layout (one layer of one 16-token block): K [16][kv_heads][head_dim]
then V [16][kv_heads][head_dim], fp16.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from . import fetch as F
from .kv import residency_version


class KVAttentionDecoder:
    # gather-mode issue policy (see _run); class-level so probes can A/B them
    issue_ahead = True      # issue K1 of layer l+1 before K5 of layer l
    timed_events = True     # timing-enabled stream events in eager steps
    overlap_layers = True   # K5 of layer l+1 starts as K5 of layer l drains (HV_ATTN_OVERLAP_PREVIOUS)
    overlap_gather = False  # the same in gather mode (measured slower, see _attend)
    balanced = False        # K5 as balanced (stream-K) ranges, one CTA per SM (HV_ATTN_BALANCED): measured slower

    def __init__(self, kv, sequences, q_heads: int, tokens: int | None = None, seed: int = 0,
                 engine: str | None = None, max_ctas: int | None = None, trace: bool = False,
                 fused: bool = False, splits: int | None = None):
        """``sequences``: sequence ids of the batch (any lengths; each attends
        over all of its tokens, or the first ``tokens`` of each when given).
        Queries are synthetic: one random fp16 query per (layer, sequence,
        q head)."""
        m = kv.m
        if q_heads % m.kv_heads:
            raise ValueError("q_heads must be a multiple of kv_heads (grouped-query attention)")
        self.kv, self.m = kv, m
        self.seqs = list(sequences)
        self.B, self.L, self.Hq = len(self.seqs), m.num_layers, q_heads
        blocks = [kv.seq_blocks[s] for s in self.seqs]
        if any(not b for b in blocks):
            raise ValueError("every sequence of the batch needs at least one block")
        lens = [sum(kv.table[bid].entries for bid in b) for b in blocks]
        self.tokens = [min(n, tokens) if tokens is not None else n for n in lens]
        self.T = max(self.tokens)
        self.ids = [bid for b in blocks for bid in b]            # sequence-major block order
        self.dev = torch.device(kv.dev)
        self.engine = engine if engine is not None else kv.engine
        # the gathers share the SMs with the attention kernels: by default the
        # K1 grid is capped (64 CTAs = 4 MiB in flight, enough for PCIe and
        # NVLink) so attention of layer l runs beside the gather of layer l+1
        self.max_ctas = 64 if max_ctas is None else max_ctas
        self.page = m.page_bytes
        self.fused = fused
        n = len(self.ids)
        self.bufs = [] if fused else [torch.empty(n * self.page, dtype=torch.uint8, device=self.dev)
                                      for _ in range(2)]
        # gather mode: the attention's page table is the gathered buffer
        self.buf_pages = [torch.arange(n, dtype=torch.int64, device=self.dev) * self.page + b.data_ptr()
                          for b in self.bufs]
        g = torch.Generator().manual_seed(seed)
        self.q = (torch.randn(self.L, self.B, q_heads, m.head_dim, generator=g)).to(torch.float16).to(self.dev)
        starts = np.concatenate([[0], np.cumsum([len(b) for b in blocks])]).astype(np.int32)
        self.seq_start = torch.from_numpy(starts).to(self.dev)
        self.seq_tokens = torch.tensor(self.tokens, dtype=torch.int32, device=self.dev)
        self.nb = max(len(b) for b in blocks)
        # flash-decoding splits: one wave of (sequence, KV head, split) CTAs,
        # one 8-warp CTA per SM.  Measured on B200 (tools/attn_probe.py, HBM
        # pages, KV GB/s): 4 x 4k: 4 splits 3,988, 8: 3,313, 19: 2,339;
        # 1 x 128k: 18 splits 5,900, 37: 5,227, 74: 4,568 -- fewer, longer
        # splits amortize the partial write and merge
        # Balanced form (opt-in, up to 256 sequences): the (sequence, KV head,
        # block) units cut into one equal range per SM, so the grid fills the
        # machine whatever pairs x splits comes to (config 1: 32 pairs -> 4
        # splits = 128 CTAs on 148 SMs in the grid form).  Measured (r5d,
        # tools/kv_decode_probe.py, in place, CUDA graph, PDL across layers):
        # 4 x 4k 6,842 vs 10,277 tok/s for the grid, 128k 330 vs 407 -- with
        # programmatic dependent launch the grid's idle SMs are where the next
        # layer's CTAs start, and its CTAs finish staggered; the balanced
        # CTAs all finish together.  Alone (tools/attn_probe.py) 26.3 vs 21.0 us
        # at 4 x 4k and 98 vs 96 us at 128k.
        sms = torch.cuda.get_device_properties(self.dev).multi_processor_count
        self.use_balanced = self.balanced and splits is None and self.B <= 256
        if self.use_balanced:
            self.splits = sms
            slots = sms + self.B * m.kv_heads
        else:
            self.splits = splits or max(1, min(self.nb, sms // (self.B * m.kv_heads)))
            slots = self.B * m.kv_heads * self.splits
        g_heads = q_heads // m.kv_heads
        self.part = torch.empty(slots * g_heads * (m.head_dim + 2), dtype=torch.float32, device=self.dev)
        self.scale = 1.0 / math.sqrt(m.head_dim)
        self.fetch_h = kv.stream
        self.fetch = torch.cuda.ExternalStream(kv.stream, device=self.dev)
        self.compute = torch.cuda.Stream(self.dev)
        self.trace = trace
        self._tr: dict = {}
        self._graph = None
        self._tab_dev = torch.empty(2, len(self.ids), dtype=torch.int64, device=self.dev)
        self._tab_version, self._tab_handles = None, []
        self._layers = torch.arange(self.L, dtype=torch.int64, device=self.dev).unsqueeze(1)

    def _upload_table(self) -> list:
        """Resolve the block table on the host and copy it (pinned, async) into
        the decoder's device table on the current stream, ordered after every
        earlier step and before this one.  Returns the peer handles read.
        Skipped while the KV residency version is unchanged (kv.residency_version:
        every tier/slot/slab change bumps it), so a steady decode step costs no
        host-side table walk."""
        ver = residency_version()
        if ver == self._tab_version:        # no block moved since the last upload
            return self._tab_handles
        bases, strides, handles = self.kv.page_table(self.ids)
        if np.any(bases % 16) or np.any(strides % 16):
            raise ValueError("paged attention reads 16-byte granules: KV pages must be 16-byte aligned")
        self._tab_host = (np.asarray(bases, dtype=np.uint64), np.asarray(strides, dtype=np.uint64))
        self._runs = {}
        tab = torch.from_numpy(np.stack([bases, strides]).view(np.int64)).pin_memory()
        self._tab_dev.copy_(tab, non_blocking=True)
        self._tab_version, self._tab_handles = ver, handles
        return handles

    def _gather_runs(self, layer: int):
        """The layer's gather as contiguous runs (host arrays: source, offset in
        the gather buffer, bytes), or None when the pages are scattered; cached
        per uploaded table."""
        if not getattr(self, "coalesce", True) or getattr(self, "_tab_host", None) is None:
            return None
        if layer not in self._runs:
            bases, strides = self._tab_host
            n = len(bases)
            off = np.arange(n, dtype=np.uint64) * np.uint64(self.page)
            r = F.layer_runs(bases + np.uint64(layer) * strides, np.zeros(n, dtype=np.uint64), off,
                             np.zeros(n, dtype=np.uint64), self.page, 1)
            self._runs[layer] = r
        return self._runs[layer]

    def _attend(self, layer: int, pages: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """hv_paged_decode_attention over the page table `pages` [n] (int64)
        into `out` [B, Hq, D] (fp32, contiguous)."""
        m = self.m
        # in place, the layers' attention kernels follow each other on the
        # compute stream and read only the step's static inputs: each one may
        # start while the previous layer's drains (programmatic dependent
        # launch).  Measured (tools/kv_decode_probe.py, r2u, CUDA graph):
        # 4 x 4k 10,299 vs 6,658 tok/s, 128k 402 vs 337.  In gather mode an
        # early attention CTA would hold SMs the next K1 gather needs (graph:
        # 1,791 vs 3,235 tok/s), so there it stays off; re-measured with the
        # K1 stream at the greatest priority (r4s): 1,792 vs 3,244, 128k 59
        # vs 108 -- priority orders dispatch, it cannot evict resident CTAs.
        flags = N.ATTN_OVERLAP_PREVIOUS if (self.overlap_layers and (self.fused or self.overlap_gather)
                                            and layer > 0) else 0
        if self.use_balanced:
            flags |= N.ATTN_BALANCED
        N.call("hv_paged_decode_attention_ex", pages.data_ptr(), self.seq_start.data_ptr(),
               self.seq_tokens.data_ptr(), self.q[layer].data_ptr(), out.data_ptr(), self.part.data_ptr(), self.B,
               self.Hq, m.kv_heads, m.head_dim, m.block_tokens, self.splits, self.scale, flags,
               torch.cuda.current_stream(self.dev).cuda_stream)
        return out

    def _run(self) -> torch.Tensor:
        """The device work of a step over the uploaded table: per-layer page
        addresses (one broadcast), then the gathers and attention (or the
        attention alone, in place).  Host-free, so it can be graph-captured."""
        cur = torch.cuda.current_stream(self.dev)
        self.fetch.wait_stream(cur)
        self.compute.wait_stream(cur)
        # allocated on the stream that writes them first; the in-place
        # attention reads them on the compute stream after a stream wait
        with torch.cuda.stream(self.fetch):
            src = self._tab_dev[0].unsqueeze(0) + self._layers * self._tab_dev[1].unsqueeze(0)
        # one output allocation per step (on the compute stream, its writer)
        with torch.cuda.stream(self.compute):
            outs = torch.empty(self.L, self.B, self.Hq, self.m.head_dim, dtype=torch.float32, device=self.dev)
        if self.fused:                      # attention straight over the resident pages
            with torch.cuda.stream(self.compute):
                self.compute.wait_stream(self.fetch)
                if not torch.cuda.is_current_stream_capturing():   # graph pools are never recycled mid-replay
                    src.record_stream(self.compute)
                for layer in range(self.L):
                    if self.trace:
                        c0 = torch.cuda.Event(enable_timing=True)
                        c0.record(self.compute)
                    self._attend(layer, src[layer], outs[layer])
                    if self.trace:
                        c1 = torch.cuda.Event(enable_timing=True)
                        c1.record(self.compute)
                        self._tr[layer] = {"fetch": (c0, c0), "compute": (c0, c1)}
        else:
            # K1 of layer l+1 and K5 of layer l become ready together (when K1
            # of layer l completes); the step overlaps them only if K1 places
            # its CTAs first, otherwise the pair serializes (128k context, K1
            # capped at 64 CTAs: 18.0 vs 10.5 ms per step).  So the gather of
            # layer l+1 is issued before the attention of layer l, and eager
            # steps record timing-enabled events, whose heavier record delays
            # K5's start (tools/event_probe.py).
            consumed = [None, None]
            got = [None] * self.L
            timed_ev = self.timed_events and not torch.cuda.is_current_stream_capturing()

            def gather(layer):
                b = layer % 2
                if consumed[b] is not None:
                    self.fetch.wait_event(consumed[b])
                if self.trace:
                    f0 = torch.cuda.Event(enable_timing=True)
                    f0.record(self.fetch)
                    self._tr[layer] = {"fetch": (f0, None)}
                runs = None if torch.cuda.is_current_stream_capturing() else self._gather_runs(layer)
                if runs is not None:
                    # the layer's pages lie in a few long contiguous runs (a
                    # sequence evicted together): the engine per source moves
                    # them -- the copy engine from the pinned host tier
                    rs, roff, rbytes = runs
                    rd = roff + np.uint64(self.bufs[b].data_ptr())
                    N.call("hv_swap_blocks_batch", rs.ctypes.data, rd.ctypes.data, rbytes.ctypes.data, len(rs),
                           N.ENGINE_AUTO, self.max_ctas, self.fetch_h)
                else:
                    F.kv_gather(src[layer], self.page, dst=self.bufs[b], engine=self.engine, max_ctas=self.max_ctas,
                                stream=self.fetch_h)
                got[layer] = torch.cuda.Event(enable_timing=timed_ev or self.trace)
                got[layer].record(self.fetch)
                if self.trace:
                    self._tr[layer]["fetch"] = (f0, got[layer])

            ahead = 1 if self.issue_ahead else 0
            for layer in range(min(ahead, self.L)):
                gather(layer)
            for layer in range(self.L):
                if layer + ahead < self.L:
                    gather(layer + ahead)
                with torch.cuda.stream(self.compute):
                    self.compute.wait_event(got[layer])
                    if self.trace:
                        c0 = torch.cuda.Event(enable_timing=True)
                        c0.record(self.compute)
                    self._attend(layer, self.buf_pages[layer % 2], outs[layer])
                    done = torch.cuda.Event(enable_timing=timed_ev or self.trace)
                    done.record(self.compute)
                    consumed[layer % 2] = done
                if self.trace:
                    self._tr[layer]["compute"] = (c0, done)
        cur.wait_stream(self.compute)
        cur.wait_stream(self.fetch)
        return outs

    def step(self) -> torch.Tensor:
        """One decode step over all layers: returns the attention outputs
        [L, B, Hq, D] (after capture_graph(), a buffer the next step reuses)."""
        from .kv import KVTier
        rt = self.kv.rt
        # a slab whose release began is drained before this step reads the
        # table (see MoEDecoder._settle_releases): the callbacks then move its
        # blocks to the host copy (Backed) or mark them lost (Lossy)
        if rt.release_epoch != getattr(self, "_release_seen", 0):
            self._release_seen = rt.release_epoch
            if any(not s.live or rt.is_draining(s.handle) for s in self.kv.slabs
                   if s.blocks and any(self.kv.table[b].tier is KVTier.PEER_HBM for b in s.blocks.values())):
                torch.cuda.synchronize(self.dev)
                self.kv.sys.loop.poll()
        if residency_version() != self._tab_version:
            lost = [bid for bid in self.ids if self.kv.table[bid].tier is KVTier.NOT_MATERIALIZED]
            if lost:                        # Lossy blocks revoked since the last step: recompute
                self.kv.reload(lost)
        handles = self._upload_table()
        batch = rt.begin_reads(handles) if handles else None
        if self._graph is not None:
            self._graph.replay()
            out = self._graph_out
        else:
            out = self._run()
        # the KV manager's later writes (evict / reload K1 on the fetch stream)
        # must follow this step's reads of the pages -- in place (fused) the
        # attention reads local, host and peer pages on the compute stream
        fin = torch.cuda.Event()
        fin.record(torch.cuda.current_stream(self.dev))
        self.fetch.wait_event(fin)
        if batch is not None:               # the drain completes when the step's reads have
            self.kv.sys.engine.track([lambda _x, bt=batch: rt.end_reads(bt)])
        return out

    def capture_graph(self) -> None:
        """Capture the device work of a step (the table broadcast, every K1
        gather and K5 attention, both streams) as one CUDA graph; each later
        step() is the table upload plus one replay."""
        if self.trace:
            raise ValueError("trace mode records per-launch events; capture without trace")
        if self._graph is not None:
            return
        self._upload_table()
        cur = torch.cuda.current_stream(self.dev)
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(cur)
        with torch.cuda.stream(side):       # warm-up outside capture (allocator, lazy attributes)
            for _ in range(2):
                self._run()
        cur.wait_stream(side)
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._graph_out = self._run()
        torch.cuda.synchronize(self.dev)
        self._graph = g

    def overlap_report(self) -> dict:
        """Device-clock gather / attention intervals of the last traced step."""
        torch.cuda.synchronize(self.dev)
        if not self._tr:
            return {}
        base = self._tr[0]["fetch"][0]
        iv = {l: {k: (base.elapsed_time(a), base.elapsed_time(b)) for k, (a, b) in v.items()}
              for l, v in self._tr.items()}
        fetch_ms = sum(v["fetch"][1] - v["fetch"][0] for v in iv.values())
        comp_ms = sum(v["compute"][1] - v["compute"][0] for v in iv.values())
        span = max(v["compute"][1] for v in iv.values())
        return {"layers": len(iv), "gather_ms": fetch_ms, "attention_ms": comp_ms, "span_ms": span,
                "serial_ms": fetch_ms + comp_ms}
