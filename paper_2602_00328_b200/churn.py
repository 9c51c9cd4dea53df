"""Dynamic donor availability (BASELINE configs[4]): churn timelines driving
mid-decode revocation and re-placement.

Reference pieces restated (the availability process is the input side of the
revocation path):
* AvailabilityProcess / markov_availability / availability_from_trace
  (traces.py:155-213) — same sampling sequence, so a seed yields the same
  timeline (tests/golden/traces.json);
* HarvestRuntime.apply_availability / _availability_step (runtime.py:465-487)
  — used as is from paper_2602_00328_b200.runtime;
* rebalance (moe.py:155-197) — re-placement once capacity returns.

``ChurnDriver`` maps a timeline (modeled seconds) onto wall time on a
DeviceLoop and re-places host-resident experts after every tick.  Revocations
that land while fetch kernels are reading a segment are drained by CUDA
events before the segment is invalidated, the callback flips the residency to
the host copy, and the VMM chunks are unmapped only after the drain.
"""
from __future__ import annotations

import random
from dataclasses import dataclass, field

from .memalloc import Tier


@dataclass
class AvailabilityProcess:
    """traces.py:155-168: piecewise-constant harvestable bytes over time."""
    steps: list = field(default_factory=list)

    def level_at(self, time: float) -> int:
        level = 0
        for t, v in self.steps:
            if t <= time:
                level = v
            else:
                break
        return level


def markov_availability(levels: list[int], mean_sojourns: list[float], seed: int,
                        horizon: float) -> AvailabilityProcess:
    """traces.py:190-213: exponential sojourns, uniform jump to another level."""
    if len(levels) != len(mean_sojourns):
        raise ValueError("levels and mean_sojourns must have equal length")
    if not levels:
        raise ValueError("need at least one level")
    if any(s <= 0 for s in mean_sojourns):
        raise ValueError("sojourn times must be positive")
    rng = random.Random(seed)
    steps, t, state = [], 0.0, 0
    while t < horizon:
        steps.append((t, levels[state]))
        t += rng.expovariate(1.0 / mean_sojourns[state])
        if len(levels) > 1:
            nxt = rng.randrange(len(levels) - 1)
            state = nxt if nxt < state else nxt + 1
    return AvailabilityProcess(steps=steps)


def availability_from_trace(utilizations: list[tuple[float, float]], capacity: int, time_scale: float = 1.0,
                            reserved: int = 0, headroom: int = 0) -> AvailabilityProcess:
    """traces.py:171-187 on (timestamp, utilization) pairs:
    harvestable = capacity*(1-u) - reserved - headroom, clamped at 0."""
    if not utilizations:
        raise ValueError("no snapshot records")
    pts = sorted(utilizations)
    t0 = pts[0][0]
    return AvailabilityProcess(steps=[((t - t0) * time_scale,
                                       max(0, int(capacity * (1.0 - u)) - reserved - headroom)) for t, u in pts])


class ChurnDriver:
    """Apply availability timelines to peer devices of a live HarvestSystem."""

    def __init__(self, system, processes: dict, time_scale: float = 1.0):
        self.sys = system
        self.rt = system.runtime
        self.processes = processes
        self.time_scale = time_scale
        self.started = False

    def start(self) -> None:
        t0 = self.sys.loop.now
        for peer_id, proc in self.processes.items():
            self.rt.apply_availability(peer_id, [(t0 + t * self.time_scale, int(lv)) for t, lv in proc.steps])
        self.started = True

    def tick(self, replace=None) -> dict:
        """Fire due availability steps / completions; then run ``replace``
        (e.g. a rebalance closure) to re-place experts on freed capacity."""
        self.sys.loop.poll()
        migrated = replace() if replace is not None else []
        self.sys.loop.poll()
        return {"revoked": len(self.sys.loop.log.of_kind("revoke_begin")), "migrated": len(migrated)}


def mem_get_info(device: int) -> tuple[int, int]:
    """(free, total) HBM bytes of a CUDA device (hv_mem_get_info)."""
    import ctypes as C

    from . import _native as N
    free, total = C.c_uint64(), C.c_uint64()
    N.call("hv_mem_get_info", device, C.byref(free), C.byref(total))
    return free.value, total.value


class DonorMonitor:
    """Real co-tenant pressure: poll each donor GPU's free HBM (cudaMemGetInfo)
    and set the runtime's availability ceiling for that peer to what the
    harvest currently holds plus what is still free, minus a safety headroom.
    A drop triggers the reference's own reclaim (runtime.py:476-487): LRU
    revocation, drained, invalidated, called back, and the VMM chunks
    unmapped so the co-tenant gets the memory."""

    def __init__(self, system, headroom: int = 1 << 30, meminfo=None):
        self.sys = system
        self.rt = system.runtime
        self.headroom = headroom
        self.meminfo = meminfo or mem_get_info
        self.last: dict[int, int] = {}

    def level(self, peer_id: int) -> int:
        pool = self.sys.pools[peer_id]
        free, _total = self.meminfo(pool.donor)
        held = pool.committed_bytes   # HBM this harvest already holds on the donor
        return max(0, int(free) + int(held) - self.headroom)

    def poll(self) -> dict:
        """Apply the current levels now; returns {peer_id: level}."""
        out = {}
        for peer_id in self.sys.pools:
            lv = min(self.level(peer_id), self.rt.devices[peer_id].spec.usable)
            if self.last.get(peer_id) != lv:
                self.rt.set_availability(peer_id, lv)
                self.last[peer_id] = lv
            out[peer_id] = lv
        self.sys.loop.poll()
        return out


def expert_tier_counts(residency) -> dict:
    c = {t.value: 0 for t in Tier}
    for e in residency.entries.values():
        c[e.tier.value] += 1
    return c
