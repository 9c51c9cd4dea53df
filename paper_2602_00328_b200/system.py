"""Assemble a real Harvest deployment on one node: compute GPU, donor pools,
pinned host tier, DeviceLoop, CudaTransferEngine and HarvestRuntime.

Device ids follow the reference's standard topology (profiles.py:152-181):
compute 0, peers 1..N, host N+1.  Link constants are the *predictions* the
Locality policy and the modeled engine use; the defaults are B200 figures
(NVLink 5 peer copy ~770 GB/s per direction, PCIe Gen5 x16 ~55 GB/s measured)
and can be refit from measurements with interconnect.calibrate.
"""
from __future__ import annotations

import torch

from . import _native as N
from .events import DeviceLoop
from .interconnect import CudaTransferEngine, LinkKind, LinkSpec, MemoryMap, Topology
from .memalloc import DeviceSpec, Tier
from .pool import HostTier, PeerPool
from .runtime import HarvestRuntime, Policy

GiB = 1 << 30
NVLINK_PEER = (2.0e-6, 770e9)   # fixed cost s, bandwidth B/s (B200_PROFILING.md peer copy)
PCIE_HOST = (10.0e-6, 55e9)     # measured pinned H2D on the B200 box (profiles/)


def build_topology(n_peers: int, peer_capacity, host_capacity: int, local_capacity: int = 180 * GiB,
                   peer_reserved: int = 0, peer_headroom: int = 0, cuda_devices=None,
                   compute_cuda: int | None = None, peer_link=NVLINK_PEER, host_link=PCIE_HOST) -> Topology:
    caps = peer_capacity if isinstance(peer_capacity, (list, tuple)) else [peer_capacity] * n_peers
    host_id = n_peers + 1
    devices = [DeviceSpec(0, Tier.LOCAL_HBM, local_capacity, cuda_device=compute_cuda)]
    links = []
    for pid in range(1, n_peers + 1):
        devices.append(DeviceSpec(pid, Tier.PEER_HBM, caps[pid - 1], reserved=peer_reserved, headroom=peer_headroom,
                                  cuda_device=None if cuda_devices is None else cuda_devices[pid - 1]))
        links.append(LinkSpec(LinkKind.PEER_LINK, peer_link[0], peer_link[1], endpoints=(0, pid)))
        links.append(LinkSpec(LinkKind.HOST_LINK, host_link[0], host_link[1], endpoints=(pid, host_id)))
    devices.append(DeviceSpec(host_id, Tier.HOST_DRAM, host_capacity))
    links.append(LinkSpec(LinkKind.HOST_LINK, host_link[0], host_link[1], endpoints=(0, host_id)))
    return Topology(devices=devices, links=links)


class HarvestSystem:
    """One compute GPU harvesting HBM from ``donors`` (CUDA device indices).

    ``donor_bytes`` is each donor's harvestable range (the DeviceSpec usable
    capacity); VMM pools commit physical memory only under live allocations,
    in ``chunk_bytes`` units.  32 MiB is the default: measured on B200, a
    17.3 MB expert costs 11.5 ms to commit in 2 MiB chunks and 0.21 ms in
    32 MiB chunks (profiles/r1_vmm_chunk_cost.json).
    ``pools`` may pass pre-built PeerPool objects instead (e.g. IPC imports
    from other processes), keyed by peer index 1..N.
    """

    def __init__(self, compute: int, donors=(), donor_bytes=0, host_bytes: int = 0, local_bytes: int = 0,
                 policy: Policy | None = None, chunk_bytes: int = 32 << 20, pool_mode: str = "vmm",
                 engine: str = "auto", max_ctas: int = 0, pools: dict | None = None,
                 peer_reserved: int = 0, peer_headroom: int = 0, host_tier: HostTier | None = None,
                 log_transfers: bool = True, stream=None):
        self.compute = compute
        torch.cuda.set_device(compute)
        self.pools: dict[int, PeerPool] = {}
        if pools:
            self.pools = dict(pools)
            donors = [p.donor for _, p in sorted(self.pools.items())]
        else:
            sizes = donor_bytes if isinstance(donor_bytes, (list, tuple)) else [donor_bytes] * len(donors)
            for i, (d, nb) in enumerate(zip(donors, sizes), start=1):
                if d != compute:
                    N.call("hv_enable_peer_access", compute, d)
                self.pools[i] = PeerPool(d, nb + peer_reserved + peer_headroom, readers=[compute],
                                         chunk_bytes=chunk_bytes, mode=pool_mode)
        self.donors = list(donors)
        n = len(self.pools)
        caps = [self.pools[i].nbytes for i in range(1, n + 1)]
        self.host = host_tier if host_tier is not None else (HostTier(host_bytes) if host_bytes else None)
        host_cap = self.host.nbytes if self.host is not None else 1
        self.local = torch.empty(max(local_bytes, 1), dtype=torch.uint8, device=f"cuda:{compute}")
        self.topology = build_topology(n, caps, host_cap, local_capacity=max(local_bytes, 1),
                                       peer_reserved=peer_reserved, peer_headroom=peer_headroom,
                                       cuda_devices=self.donors, compute_cuda=compute)
        self.host_id = n + 1
        self.memory = MemoryMap()
        self.memory.register(0, self.local.data_ptr(), self.local.numel())
        for i, p in self.pools.items():
            self.memory.register(i, p.va, p.nbytes)
        if self.host is not None:
            self.memory.register(self.host_id, self.host.d_alias, self.host.nbytes)
        self.loop = DeviceLoop()
        # the fetch stream is the most urgent on the device: a decode step's
        # next fetch must not wait behind the compute stream's CTAs
        self.engine = CudaTransferEngine(self.loop, self.topology, self.memory, compute, stream=stream,
                                         engine=engine, max_ctas=max_ctas, log_transfers=log_transfers,
                                         priority="urgent")
        self.runtime = HarvestRuntime(self.loop, self.topology, policy, compute_device_id=0,
                                      engine=self.engine, pools=self.pools)
        # placement copy-ins (K3, rebalance) run on their own stream so they
        # share the links with, but never queue behind, the fetch stream
        self.placement_engine = CudaTransferEngine(self.loop, self.topology, self.memory, compute,
                                                   engine=engine, max_ctas=max_ctas, log_transfers=log_transfers)
        self.runtime.placement_engine = self.placement_engine

    def close(self) -> None:
        self.loop.run()
        self.engine.close()
        self.placement_engine.close()
        for p in self.pools.values():
            p.close()
        if self.host is not None:
            self.host.close()
