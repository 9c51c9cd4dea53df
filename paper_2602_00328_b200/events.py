"""Event loops and the event log of the B200 Harvest runtime.

The reference drives everything from one deterministic discrete-event loop
(events.py:61-103): a heap keyed by (time, seq) plus an append-only EventLog
whose records carry strictly increasing (time, seq) stamps (events.py:16-58).
The B200 runtime keeps that log format — so the reference's own checkers
(verify.py:25-88) run unchanged on logs of real GPU runs — and offers two loops:

* ``VirtualLoop``  the reference semantics exactly (modeled time).  Used with
                   the modeled transfer engine for planning, deterministic
                   replay and the CPU test tier.
* ``DeviceLoop``   wall-clock time; deferred callbacks run when due and
                   transfer completions are discovered by polling CUDA events
                   (the real "drain", runtime.py:345-356).  Callbacks always run
                   on the caller's thread inside poll()/run(), never on a CUDA
                   host-function thread, preserving runtime.py:403-405.
"""
from __future__ import annotations

import heapq
import itertools
import time
from dataclasses import dataclass, field


@dataclass(frozen=True)
class LogRecord:
    """events.py:16-31."""
    time: float
    seq: int
    kind: str
    data: dict = field(default_factory=dict, compare=False)

    @property
    def stamp(self) -> tuple[float, int]:
        return (self.time, self.seq)

    def __repr__(self) -> str:
        fields = " ".join(f"{k}={v}" for k, v in sorted(self.data.items()))
        return f"[t={self.time:.9f} #{self.seq}] {self.kind} {fields}"


class EventLog:
    """events.py:34-58."""

    def __init__(self, enabled: bool = True):
        self.records: list[LogRecord] = []
        self.enabled = enabled

    def append(self, time_: float, seq: int, kind: str, **data) -> LogRecord:
        rec = LogRecord(time_, seq, kind, data)
        if self.enabled:
            self.records.append(rec)
        return rec

    def of_kind(self, *kinds: str) -> list[LogRecord]:
        want = set(kinds)
        return [r for r in self.records if r.kind in want]

    def __len__(self) -> int:
        return len(self.records)

    def __iter__(self):
        return iter(self.records)

    def excerpt(self, center_seq: int, radius: int = 6) -> str:
        return "\n".join(repr(r) for r in self.records if abs(r.seq - center_seq) <= radius)


class _LoopBase:
    wall_clock = False

    def __init__(self):
        self._queue: list[tuple[float, int, tuple]] = []
        self._counter = itertools.count()
        self.log = EventLog()
        self._pollers: list = []

    def next_seq(self) -> int:
        return next(self._counter)

    def schedule(self, delay: float, fn, *args) -> int:
        if delay < 0:
            raise ValueError(f"negative delay {delay}")
        return self._push(self.now + delay, fn, args)

    def schedule_at(self, t: float, fn, *args) -> int:
        now = self.now
        if t < now:
            if not self.wall_clock:
                raise ValueError(f"cannot schedule at {t} before now {now}")
            t = now  # wall time moved on between computing t and this call
        return self._push(t, fn, args)

    def _push(self, t: float, fn, args) -> int:
        seq = self.next_seq()
        heapq.heappush(self._queue, (t, seq, (fn, args)))
        return seq

    def record(self, kind: str, **data) -> LogRecord:
        return self.log.append(self.now, self.next_seq(), kind, **data)

    def pending(self) -> int:
        return len(self._queue) + sum(p.pending() for p in self._pollers)

    def add_poller(self, poller) -> None:
        """A poller exposes poll(loop) -> int (completions fired), pending(),
        and wait_one() (block until at least one completion is observable)."""
        self._pollers.append(poller)


class VirtualLoop(_LoopBase):
    """events.Simulator semantics (events.py:61-103): modeled time only."""

    def __init__(self, start_time: float = 0.0):
        super().__init__()
        self.now = start_time

    def run(self, until: float | None = None) -> None:
        while self._queue:
            t, _seq, (fn, args) = self._queue[0]
            if until is not None and t > until:
                break
            heapq.heappop(self._queue)
            self.now = t
            fn(*args)
        if until is not None and until > self.now:
            self.now = until


class DeviceLoop(_LoopBase):
    """Wall-clock loop.  ``now`` is seconds since construction."""

    wall_clock = True

    def __init__(self):
        super().__init__()
        self._t0 = time.perf_counter()

    @property
    def now(self) -> float:
        return time.perf_counter() - self._t0

    def poll(self) -> int:
        """Fire due deferred callbacks and observed transfer completions."""
        fired = 0
        progress = True
        while progress:
            progress = False
            for p in self._pollers:
                n = p.poll(self)
                fired += n
                progress |= n > 0
            now = self.now
            while self._queue and self._queue[0][0] <= now:
                _t, _seq, (fn, args) = heapq.heappop(self._queue)
                fn(*args)
                fired += 1
                progress = True
        return fired

    def run(self, until: float | None = None) -> None:
        """Process until nothing is pending (or wall time `until`)."""
        while True:
            self.poll()
            if until is not None and self.now >= until:
                return
            busy = [p for p in self._pollers if p.pending()]
            if busy:
                busy[0].wait_one()
                continue
            if not self._queue:
                return
            delay = self._queue[0][0] - self.now
            if until is not None:
                delay = min(delay, until - self.now)
            if delay > 0:
                time.sleep(delay)
