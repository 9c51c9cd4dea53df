"""Links, topology and transfer engines.

API kept from the reference (interconnect.py:21-221): LinkKind, LinkSpec,
transfer_time, Topology, TransferRequest, Transfer, RoutingError,
CalibrationError, calibrate, calibration_rms, load_calibration_points.

Two engines implement ``schedule_transfer(req, on_complete, initiator,
handle_key)`` (interconnect.py:133-165):

* ``ModeledTransferEngine`` — the reference's affine-cost, per-pair FIFO model
  (fixed_cost + size/bandwidth, interconnect.py:51-54, :147-150) on a
  VirtualLoop.  It is the planner/predictor, and the engine under the CPU
  tier's deterministic replay of the reference's decisions.
* ``CudaTransferEngine`` — real copies.  Every batch of requests becomes ONE
  launch of the sm_100a batched-fetch kernel (K2; K1 for uniform pages) on
  the engine's fetch stream, followed by one CUDA event.  Completion is
  discovered by the DeviceLoop polling that event; then transfer_complete is
  logged and the callbacks fire in issue order (the drain).  Unlike the model,
  transfers are not serialized per device pair: every object of a batch is in
  flight at once and NVLink is full duplex.
"""
from __future__ import annotations

import ctypes as C
import os
import enum
import math
from collections import deque
from dataclasses import dataclass, field
from typing import Iterable, TextIO

import numpy as np

from . import _native as N
from .memalloc import DeviceSpec, Segment, Tier


class LinkKind(enum.Enum):
    PEER_LINK = "PeerLink"
    HOST_LINK = "HostLink"


class CalibrationError(Exception):
    pass


class RoutingError(Exception):
    pass


@dataclass(frozen=True)
class LinkSpec:
    """interconnect.py:34-48."""
    kind: LinkKind
    fixed_cost: float
    bandwidth: float
    endpoints: tuple[int, int]
    hops: int = 1

    def __post_init__(self):
        if self.fixed_cost < 0:
            raise ValueError("fixed_cost must be >= 0")
        if self.bandwidth <= 0:
            raise ValueError("bandwidth must be > 0")
        if self.hops < 1:
            raise ValueError("hops must be >= 1")


def transfer_time(link: LinkSpec, size: int) -> float:
    """interconnect.py:51-54."""
    if size < 0:
        raise ValueError("size must be >= 0")
    return link.fixed_cost + size / link.bandwidth


@dataclass
class Topology:
    """interconnect.py:57-100: every peer and the host must link to each
    compute device; at most one link per device pair."""
    devices: list[DeviceSpec]
    links: list[LinkSpec]
    _by_pair: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        ids = [d.device_id for d in self.devices]
        if len(set(ids)) != len(ids):
            raise ValueError("duplicate device ids in topology")
        for link in self.links:
            pair = frozenset(link.endpoints)
            if len(pair) != 2:
                raise ValueError(f"link endpoints must differ: {link.endpoints}")
            if pair in self._by_pair:
                raise ValueError(f"more than one link between {link.endpoints}")
            self._by_pair[pair] = link
        for local in (d for d in self.devices if d.tier == Tier.LOCAL_HBM):
            for dev in self.devices:
                if dev.tier in (Tier.PEER_HBM, Tier.HOST_DRAM) and self.link_between(local.device_id, dev.device_id) is None:
                    raise ValueError(f"device {dev.device_id} ({dev.tier.value}) not linked to compute device {local.device_id}")

    def device(self, device_id: int) -> DeviceSpec:
        for d in self.devices:
            if d.device_id == device_id:
                return d
        raise KeyError(f"unknown device id {device_id}")

    def link_between(self, a: int, b: int) -> LinkSpec | None:
        return self._by_pair.get(frozenset((a, b)))

    def hops_between(self, a: int, b: int) -> int:
        link = self.link_between(a, b)
        if link is None:
            raise RoutingError(f"no link between devices {a} and {b}")
        return link.hops


@dataclass(frozen=True)
class TransferRequest:
    """interconnect.py:103-113."""
    src: tuple[int, Segment]
    dst: tuple[int, Segment]
    size: int
    issue_time: float
    tag: object = None

    def __post_init__(self):
        if self.src[1].size != self.size or self.dst[1].size != self.size:
            raise ValueError("src/dst segment sizes must equal transfer size")


@dataclass
class Transfer:
    """interconnect.py:116-122 (completion_time is filled in when observed
    for real transfers)."""
    request: TransferRequest
    link: LinkSpec | None
    start_time: float
    completion_time: float | None
    seq: int


class ModeledTransferEngine:
    """interconnect.TransferEngine (interconnect.py:125-165) restated."""

    def __init__(self, loop, topology: Topology):
        self.sim = loop
        self.topology = topology
        self._busy_until: dict[frozenset, float] = {}

    def schedule_transfer(self, req: TransferRequest, on_complete=None, initiator: str = "app",
                          handle_key: tuple | None = None) -> Transfer:
        src_dev, dst_dev = req.src[0], req.dst[0]
        link = self.topology.link_between(src_dev, dst_dev)
        if link is None:
            raise RoutingError(f"no link between devices {src_dev} and {dst_dev}")
        if req.issue_time < self.sim.now:
            raise ValueError("cannot issue a transfer in the past")
        pair = frozenset((src_dev, dst_dev))
        start = max(req.issue_time, self._busy_until.get(pair, 0.0))
        completion = start + transfer_time(link, req.size)
        self._busy_until[pair] = completion
        fields = dict(src=src_dev, dst=dst_dev, size=req.size, tag=req.tag, src_base=req.src[1].base,
                      dst_base=req.dst[1].base, initiator=initiator, handle=handle_key)
        seq = self.sim.record("transfer_start", start=start, **fields).seq
        xfer = Transfer(req, link, start, completion, seq)

        def _complete():
            self.sim.record("transfer_complete", **fields)
            if on_complete is not None:
                on_complete(xfer)

        self.sim.schedule_at(completion, _complete)
        return xfer

    def schedule_batch(self, reqs, on_completes, initiator="app", handle_keys=None):
        handle_keys = handle_keys or [None] * len(reqs)
        return [self.schedule_transfer(r, cb, initiator, hk) for r, cb, hk in zip(reqs, on_completes, handle_keys)]


class MemoryMap:
    """Topology device id -> device-visible base address of its memory:
    peer pool VA, host tier device alias, or a local arena."""

    def __init__(self):
        self._spaces: dict[int, tuple[int, int]] = {}

    def register(self, device_id: int, base: int, nbytes: int) -> None:
        self._spaces[device_id] = (base, nbytes)

    def address(self, device_id: int, seg: Segment) -> int:
        try:
            base, nbytes = self._spaces[device_id]
        except KeyError:
            raise RoutingError(f"device {device_id} has no registered memory") from None
        if seg.end > nbytes:
            raise ValueError(f"segment {seg} outside device {device_id} memory ({nbytes} bytes)")
        return base + seg.base

    def base(self, device_id: int) -> int:
        return self._spaces[device_id][0]

    def __contains__(self, device_id: int) -> bool:
        return device_id in self._spaces


class CudaTransferEngine:
    """Real batched transfers on a CUDA stream, completions via events."""

    def __init__(self, loop, topology: Topology, memory: MemoryMap, cuda_device: int,
                 stream=None, engine: str = "auto", max_ctas: int = 0, log_transfers: bool = True,
                 priority: int | str = 0):
        """``priority``: CUDA priority of the engine's own stream: an int, or
        "urgent" for the device's greatest (the decode fetch stream: its CTAs
        are dispatched ahead of the compute stream's as SMs free up, measured
        2.2x on a staged decode step, profiles/r2_priority_probe.json).  The
        HV_FETCH_PRIORITY environment value overrides "urgent" (A/B runs)."""
        self.sim = loop
        self.topology = topology
        self.memory = memory
        self.cuda_device = cuda_device
        self.engine = N.ENGINES[engine] if isinstance(engine, str) else engine
        self.max_ctas = max_ctas
        self.log_transfers = log_transfers
        self._own_stream = stream is None
        if stream is None:
            s = C.c_void_p()
            if priority == "urgent":
                priority = os.environ.get("HV_FETCH_PRIORITY")
                if priority is None:
                    least, greatest = C.c_int(), C.c_int()
                    N.call("hv_stream_priority_range", cuda_device, C.byref(least), C.byref(greatest))
                    priority = greatest.value
            N.call("hv_stream_create", cuda_device, int(priority), C.byref(s))
            self.stream = s.value or 0
        else:
            self.stream = N.stream_handle(stream)
        self._pending: deque = deque()   # (event, [(xfer, cb, fields)])
        self._free_events: list = []
        self.batches = 0
        loop.add_poller(self)

    # -- events
    def _event(self):
        if self._free_events:
            return self._free_events.pop()
        e = C.c_void_p()
        N.call("hv_event_create", self.cuda_device, 0, C.byref(e))
        return e

    def schedule_transfer(self, req: TransferRequest, on_complete=None, initiator: str = "app",
                          handle_key: tuple | None = None) -> Transfer:
        return self.schedule_batch([req], [on_complete], initiator, [handle_key])[0]

    def schedule_batch(self, reqs, on_completes, initiator: str = "app", handle_keys=None):
        n = len(reqs)
        if n == 0:
            return []
        handle_keys = handle_keys or [None] * n
        src = np.empty(n, dtype=np.uint64)
        dst = np.empty(n, dtype=np.uint64)
        size = np.empty(n, dtype=np.uint64)
        for i, r in enumerate(reqs):
            if self.topology.link_between(r.src[0], r.dst[0]) is None:
                raise RoutingError(f"no link between devices {r.src[0]} and {r.dst[0]}")
            src[i] = self.memory.address(r.src[0], r.src[1])
            dst[i] = self.memory.address(r.dst[0], r.dst[1])
            size[i] = r.size
        return self.launch_raw(src, dst, size, reqs, on_completes, initiator, handle_keys)

    def launch_raw(self, src: np.ndarray, dst: np.ndarray, size: np.ndarray, reqs=None,
                   on_completes=None, initiator: str = "app", handle_keys=None, callbacks=()):
        """Launch one batched fetch over raw device addresses (host arrays).
        Each of ``callbacks`` is called with None when the batch completes;
        the batch's event is left in ``self.last_event`` until it is polled."""
        n = len(src)
        N.call("hv_swap_blocks_batch", src.ctypes.data, dst.ctypes.data, size.ctypes.data, n,
               self.engine, self.max_ctas, self.stream)
        ev = self._event()
        N.call("hv_event_record", ev, self.stream)
        self.batches += 1
        now = self.sim.now
        items = []
        if reqs is not None:
            for i, r in enumerate(reqs):
                fields = dict(src=r.src[0], dst=r.dst[0], size=r.size, tag=r.tag, src_base=r.src[1].base,
                              dst_base=r.dst[1].base, initiator=initiator,
                              handle=handle_keys[i] if handle_keys else None)
                seq = self.sim.record("transfer_start", start=now, **fields).seq if self.log_transfers else -1
                xfer = Transfer(r, self.topology.link_between(r.src[0], r.dst[0]), now, None, seq)
                items.append((xfer, on_completes[i] if on_completes else None, fields))
        xfers = [x for x, _, _ in items]
        items.extend((None, cb, None) for cb in callbacks)
        self._pending.append((ev, items))
        self.last_event = ev
        return xfers

    def launch_raw_checked(self, src: np.ndarray, dst: np.ndarray, size: np.ndarray, expected: np.ndarray,
                           d_scratch: int, d_flags: int, d_errors: int, callbacks=()):
        """launch_raw plus the per-fetch content check fused into the same
        pass (hv_swap_blocks_batch_checked): the digest of every arrival is
        compared with ``expected`` and mismatches are added to *d_errors."""
        n = len(src)
        N.call("hv_swap_blocks_batch_checked", src.ctypes.data, dst.ctypes.data, size.ctypes.data,
               expected.ctypes.data, n, self.engine, self.max_ctas, d_scratch, d_flags, d_errors, self.stream)
        return self.track(callbacks)

    def launch_pages(self, src_page_ptrs_dev: int, n_pages: int, page_bytes: int, dst_base: int = 0,
                     dst_page_ptrs_dev: int = 0, callbacks=()):
        """K1 over device-resident page-pointer arrays; one event for the batch."""
        N.call("hv_kv_gather", src_page_ptrs_dev, dst_page_ptrs_dev, dst_base, n_pages, page_bytes,
               self.engine, self.max_ctas, self.stream)
        ev = self._event()
        N.call("hv_event_record", ev, self.stream)
        self.batches += 1
        self._pending.append((ev, [(None, cb, None) for cb in callbacks]))
        return ev

    def track(self, callbacks=()):
        """Record an event after whatever was just enqueued on the fetch stream
        (e.g. a device-descriptor launch) and run ``callbacks`` when it completes."""
        ev = self._event()
        N.call("hv_event_record", ev, self.stream)
        self._pending.append((ev, [(None, cb, None) for cb in callbacks]))
        self.last_event = ev
        return ev

    # -- poller protocol (DeviceLoop)
    def pending(self) -> int:
        return len(self._pending)

    def poll(self, loop) -> int:
        fired = 0
        done = C.c_int(0)
        while self._pending:
            ev, items = self._pending[0]
            N.call("hv_event_query", ev, C.byref(done))
            if not done.value:
                break
            self._pending.popleft()
            self._free_events.append(ev)
            now = self.sim.now
            for xfer, cb, fields in items:
                if xfer is not None:
                    xfer.completion_time = now
                    if self.log_transfers:
                        self.sim.record("transfer_complete", **fields)
                if cb is not None:
                    cb(xfer)
                fired += 1
            fired += 0 if items else 1
        return fired

    def wait_one(self) -> None:
        if self._pending:
            N.call("hv_event_synchronize", self._pending[0][0])

    def synchronize(self) -> None:
        N.call("hv_stream_synchronize", self.stream)

    def close(self) -> None:
        for ev, _ in self._pending:
            N.lib().hv_event_synchronize(ev)
        for ev in self._free_events:
            N.lib().hv_event_destroy(ev)
        self._free_events = []
        if self._own_stream and self.stream:
            N.lib().hv_stream_destroy(self.stream)
            self.stream = 0


def calibrate(points: Iterable[tuple[float, float]]) -> tuple[float, float]:
    """interconnect.py:168-188: least-squares latency = fixed + size/bandwidth."""
    pts = [(float(s), float(l)) for s, l in points]
    if len(pts) < 2:
        raise CalibrationError("need at least 2 calibration points")
    sizes = np.array([p[0] for p in pts])
    lats = np.array([p[1] for p in pts])
    if np.any(lats <= 0):
        raise CalibrationError("latencies must be positive")
    if np.all(sizes == sizes[0]):
        raise CalibrationError("all sizes equal; slope is unconstrained")
    slope, intercept = np.polyfit(sizes, lats, 1)
    if slope <= 0:
        raise CalibrationError("fitted bandwidth is not positive")
    return max(0.0, float(intercept)), 1.0 / float(slope)


def calibration_rms(points, fixed_cost: float, bandwidth: float) -> float:
    """interconnect.py:191-200."""
    errs = [((fixed_cost + s / bandwidth) - l) / l for s, l in points]
    if not errs:
        raise CalibrationError("no points")
    return math.sqrt(sum(e * e for e in errs) / len(errs))


def load_calibration_points(stream: TextIO) -> list[tuple[float, float]]:
    """interconnect.py:203-221."""
    points = []
    for lineno, raw in enumerate(stream, start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        parts = [p.strip() for p in line.split(",")]
        if len(parts) != 2:
            raise CalibrationError(f"line {lineno}: expected 2 columns, got {len(parts)}")
        try:
            size, lat = float(parts[0]), float(parts[1])
        except ValueError as exc:
            raise CalibrationError(f"line {lineno}: {exc}") from None
        points.append((size, lat))
    return points
