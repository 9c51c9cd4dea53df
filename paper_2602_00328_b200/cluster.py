"""Node layout of one-process-per-GPU Harvest: who donates to whom, where each
reader's section of a donor slab lies, which donor an expert prefers, and the
rank-group plumbing (barrier, max over ranks, rank-0 decisions).

The reference models a single compute device (runtime.py:130-133) whose
runtime places objects on peer devices 1..N (profiles.py:152-181).  On an
8-GPU node every rank is such a compute device and also donates HBM to the
others (or, for config 5, ranks are split into compute and donor roles):

- each donor exports ONE cudaIpc slab; it is cut into equal sections, one per
  reader, so readers never contend for a donor's allocator
  (``DonorLayout.section``);
- inside its section a reader's own runtime allocates with the reference's
  best fit (memalloc.py:90-114), seeing donor d as its peer index
  ``layout.peer_index(rank, d)`` (1..n_donors, the reference's device ids);
- placement prefers donors round-robin over (layer, expert), offset by rank
  (``preferred_peer``), the reference's ``preferred_devices`` hint
  (runtime.py:205-214): every layer spans every donor, and ranks walking the
  same expert index in lockstep prefer different donors.

No data-path collective exists; the process group carries
handle exchange, barriers, the max-over-ranks time and rank-0 decisions only.
Nothing here touches CUDA, so the whole layout is testable on CPU with gloo
(tests/test_cluster_gloo.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class DonorLayout:
    """Roles and slab sections of a node of ``world`` ranks.

    ``compute`` ranks read; ``donors`` export slabs.  The default (every rank
    both computes and donates to the N-1 others) is the symmetric layout of
    configs 2-4; ``split_roles`` gives config 5's asymmetric one.
    """
    world: int
    per_reader: int
    compute: tuple = ()
    donors: tuple = ()

    def __post_init__(self):
        if self.world < 1 or self.per_reader < 0:
            raise ValueError("world >= 1 and per_reader >= 0 required")
        if not self.compute:
            object.__setattr__(self, "compute", tuple(range(self.world)))
        if not self.donors:
            object.__setattr__(self, "donors", tuple(range(self.world)))
        for r in self.compute + self.donors:
            if not 0 <= r < self.world:
                raise ValueError(f"rank {r} outside world {self.world}")

    @classmethod
    def symmetric(cls, world: int, per_reader: int) -> "DonorLayout":
        return cls(world, per_reader)

    @classmethod
    def split_roles(cls, world: int, per_reader: int) -> "DonorLayout":
        """Config 5: ranks [0, N/2) are memory-pressured compute GPUs, [N/2, N) donate."""
        if world < 2:
            raise ValueError("split roles need at least 2 ranks")
        h = world // 2
        return cls(world, per_reader, tuple(range(h)), tuple(range(h, world)))

    def readers_of(self, donor: int) -> list[int]:
        """Ranks that read donor ``donor``'s slab, in section order (never the donor itself)."""
        return [r for r in self.compute if r != donor]

    def donors_of(self, reader: int) -> list[int]:
        """Donor ranks a reader harvests from, in peer-index order (peer i = donors_of[i-1])."""
        return [d for d in self.donors if d != reader]

    def slab_bytes(self, donor: int) -> int:
        return self.per_reader * len(self.readers_of(donor))

    def section(self, donor: int, reader: int) -> tuple[int, int]:
        """(offset, size) of ``reader``'s section inside ``donor``'s slab."""
        readers = self.readers_of(donor)
        if reader not in readers:
            raise ValueError(f"rank {reader} does not read donor {donor}")
        return readers.index(reader) * self.per_reader, self.per_reader

    def peer_index(self, reader: int, donor: int) -> int:
        """The runtime device id (1..n) under which ``reader`` sees ``donor``."""
        return self.donors_of(reader).index(donor) + 1


def per_reader_bytes(n_objects: int, object_bytes: int, n_donors: int, extra: int = 0) -> int:
    """Section size that holds ceil(n_objects / n_donors) objects (+ ``extra``) per donor."""
    if n_donors < 1:
        raise ValueError("at least one donor")
    return math.ceil(n_objects / n_donors) * object_bytes + extra


def preferred_peer(layer: int, expert: int, num_experts: int, rank: int, n_donors: int) -> int:
    """Round-robin donor preference (1-based peer index) for expert (layer, expert).

    Consecutive experts of a layer go to consecutive donors, so a stage's
    fetch spans all of them; the rank offset makes (k + r) mod n a permutation
    over ranks for a fixed k, so lockstep readers prefer different donors.
    """
    if n_donors < 1:
        raise ValueError("at least one donor")
    return 1 + (layer * num_experts + expert + rank) % n_donors


def place_experts(runtime, model, residency, rank: int, n_donors: int, client_id: str = "moe"):
    """Place every expert of ``model`` on the peers with the runtime's own
    harvest_alloc (runtime.py:198-235), Backed (the host copy stays
    authoritative), preferring ``preferred_peer``; record PEER residency.

    Returns (handles, seeds) in (layer, expert) order.  Raises RuntimeError
    on NoCapacity: the sections are sized to hold every expert.
    """
    from .memalloc import Tier
    from .moe import expert_content
    from .runtime import AllocationHints, Durability
    L, E, S = model.num_layers, model.num_experts, model.expert_size
    handles, seeds = [], []
    for layer in range(L):
        for e in range(E):
            pref = [preferred_peer(layer, e, E, rank, n_donors)]
            h = runtime.harvest_alloc(S, AllocationHints(preferred_devices=pref, durability=Durability.BACKED,
                                                         client_id=client_id))
            if h is None:
                raise RuntimeError(f"donor capacity exhausted at expert ({layer}, {e})")
            seed = expert_content(model, layer, e)
            runtime.set_tag(h, ("expert", layer, e))
            runtime.write_peer(h, ("expert", layer, e), seed)
            residency.set_tier(layer, e, Tier.PEER_HBM, h)
            handles.append(h)
            seeds.append(seed)
    return handles, seeds


class RankGroup:
    """The process-group plumbing every multi-rank phase uses.  With one rank
    (or no initialized group) every operation is a local no-op, so single-GPU
    code paths call the same methods."""

    def __init__(self, world: int = 1, rank: int = 0, device=None):
        self.world, self.rank = world, rank
        self.device = device   # tensors of device collectives (NCCL); None = CPU (gloo)
        self._dist = None
        if world > 1:
            import torch.distributed as dist
            if not dist.is_initialized():
                raise RuntimeError("RankGroup(world > 1) needs an initialized process group")
            self._dist = dist

    def barrier(self) -> None:
        if self._dist is not None:
            self._dist.barrier()

    def max(self, x: float) -> float:
        if self._dist is None:
            return x
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64, device=self.device or "cpu")
        self._dist.all_reduce(t, op=self._dist.ReduceOp.MAX)
        return float(t.item())

    def min(self, x: float) -> float:
        return -self.max(-x)

    def all_gather(self, obj) -> list:
        if self._dist is None:
            return [obj]
        out = [None] * self.world
        self._dist.all_gather_object(out, obj)
        return out

    def decide(self, obj, src: int = 0):
        """Rank ``src``'s value on every rank (e.g. the autotuned engine)."""
        if self._dist is None:
            return obj
        box = [obj]
        self._dist.broadcast_object_list(box, src=src)
        return box[0]

    def any(self, flag: bool) -> bool:
        return any(bool(f) for f in self.all_gather(bool(flag)))
