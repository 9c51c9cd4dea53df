"""Per-donor segment accounting — the reference's memalloc API over the native
best-fit allocator (hv_seg_*, csrc/hv_segalloc.cpp).

Same names, arguments, decisions and errors as memalloc.py:14-159: best fit by
(leftover, base), base-sorted eagerly-coalesced free list, DoubleFreeError on
unknown segments.  The reference scans the whole free list per allocation and
sums every allocation to answer allocated_bytes (memalloc.py:86-114); the
native index answers both in O(log n) / O(1).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

from . import _native as N


class Tier(enum.Enum):
    LOCAL_HBM = "LocalHBM"
    PEER_HBM = "PeerHBM"
    HOST_DRAM = "HostDRAM"


class DoubleFreeError(Exception):
    """Freeing a segment that is not currently allocated (memalloc.py:20-21)."""


@dataclass(frozen=True)
class DeviceSpec:
    """memalloc.py:24-45.  ``cuda_device`` names the physical GPU backing a
    LOCAL/PEER device (None for host or modeled-only devices)."""
    device_id: int
    tier: Tier
    capacity: int
    reserved: int = 0
    headroom: int = 0
    cuda_device: int | None = None

    def validate(self) -> None:
        if self.capacity <= 0:
            raise ValueError(f"device {self.device_id}: capacity must be > 0")
        if self.reserved < 0 or self.headroom < 0:
            raise ValueError(f"device {self.device_id}: negative reservation")
        if self.reserved + self.headroom > self.capacity:
            raise ValueError(
                f"device {self.device_id}: reserved ({self.reserved}) + "
                f"headroom ({self.headroom}) exceeds capacity ({self.capacity})")

    @property
    def usable(self) -> int:
        return self.capacity - self.reserved - self.headroom


@dataclass(frozen=True)
class Segment:
    """memalloc.py:48-64."""
    base: int
    size: int

    def __post_init__(self):
        if self.size <= 0:
            raise ValueError(f"segment size must be > 0, got {self.size}")
        if self.base < 0:
            raise ValueError(f"segment base must be >= 0, got {self.base}")

    @property
    def end(self) -> int:
        return self.base + self.size

    def overlaps(self, other: "Segment") -> bool:
        return self.base < other.end and other.base < self.end


class DeviceState:
    """memalloc.DeviceState (memalloc.py:67-71) backed by a native hv_seg."""

    def __init__(self, spec: DeviceSpec):
        self.spec = spec
        self._h = C.c_void_p()
        N.call("hv_seg_create", max(0, spec.usable), C.byref(self._h))

    def __del__(self):
        try:
            if self._h:
                N.lib().hv_seg_destroy(self._h)
        except Exception:
            pass

    @property
    def free_list(self) -> list[Segment]:
        n = C.c_uint64(0)
        N.call("hv_seg_free_list", self._h, None, C.byref(n))
        if n.value == 0:
            return []
        buf = (C.c_uint64 * (2 * n.value))()
        N.call("hv_seg_free_list", self._h, buf, C.byref(n))
        return [Segment(buf[2 * i], buf[2 * i + 1]) for i in range(n.value)]

    @property
    def allocated_bytes(self) -> int:
        v = C.c_uint64()
        N.call("hv_seg_allocated_bytes", self._h, C.byref(v))
        return v.value

    @property
    def free_bytes(self) -> int:
        v = C.c_uint64()
        N.call("hv_seg_free_bytes", self._h, C.byref(v))
        return v.value

    def probe(self, size: int) -> tuple[int, int] | None:
        """(leftover, base) of the segment a best-fit allocation would take."""
        lo, b = C.c_uint64(), C.c_uint64()
        st = N.lib().hv_seg_probe(self._h, size, C.byref(lo), C.byref(b))
        if st == N.HV_E_NOCAPACITY:
            return None
        N.check(st, "hv_seg_probe")
        return lo.value, b.value


def init_device(spec: DeviceSpec) -> DeviceState:
    """memalloc.py:74-79."""
    spec.validate()
    return DeviceState(spec)


def harvestable_capacity(state: DeviceState) -> int:
    """memalloc.py:82-83."""
    return state.free_bytes


def allocated_bytes(state: DeviceState) -> int:
    """memalloc.py:86-87."""
    return state.allocated_bytes


def alloc_best_fit(state: DeviceState, size: int) -> Segment | None:
    """memalloc.py:90-114: smallest leftover, ties to the lowest base; None
    when nothing fits."""
    if size <= 0:
        raise ValueError(f"allocation size must be > 0, got {size}")
    base = C.c_uint64()
    st = N.lib().hv_seg_alloc(state._h, size, C.byref(base))
    if st == N.HV_E_NOCAPACITY:
        return None
    N.check(st, "hv_seg_alloc")
    return Segment(base.value, size)


def free_segment(state: DeviceState, segment: Segment) -> None:
    """memalloc.py:117-138."""
    st = N.lib().hv_seg_free(state._h, segment.base, segment.size)
    if st == N.HV_E_DOUBLEFREE:
        raise DoubleFreeError(f"segment base={segment.base} size={segment.size} is not allocated")
    N.check(st, "hv_seg_free")


def check_invariants(state: DeviceState) -> None:
    """memalloc.py:141-159 (raises AssertionError on violation)."""
    if N.lib().hv_seg_check(state._h) != N.HV_OK:
        raise AssertionError(f"segment accounting invariant violated on device {state.spec.device_id}")
