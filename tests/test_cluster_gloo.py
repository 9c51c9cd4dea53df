"""Multi-rank host logic of the N>1 path on CPU (gloo, world 2 and 4).

Every rank runs the placement a GPU rank of bench.py runs -- DonorLayout
sections, a runtime over its N-1 donor sections, place_experts with the
rank-offset round-robin preference -- on a modeled runtime (no CUDA), and the
rank group's handle exchange / max / rank-0 decision.  The gathered
placements are then checked across ranks: no two readers' objects overlap
inside any donor slab, each reader stays inside its own section, every expert
is placed, every donor carries an equal share, and lockstep readers prefer
different donors at the same expert index.
"""
import os
import socket

import pytest

from paper_2602_00328_b200.cluster import DonorLayout, per_reader_bytes, preferred_peer
from paper_2602_00328_b200.moe import MoEProfile

MODEL = MoEProfile("cluster-test", num_layers=3, num_experts=10, top_k=2, expert_size=4096)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _overlaps(intervals):
    iv = sorted(intervals)
    return any(a1 > b0 for (b0, _b1), (_a0, a1) in zip(iv[1:], iv[:-1]))


# ---- single-process checks of the layout arithmetic

@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_symmetric_sections_tile_each_slab(world):
    lay = DonorLayout.symmetric(world, 1000)
    for d in range(world):
        secs = sorted(lay.section(d, r) for r in lay.readers_of(d))
        assert d not in lay.readers_of(d)
        assert [o for o, _ in secs] == [i * 1000 for i in range(world - 1)]
        assert lay.slab_bytes(d) == 1000 * (world - 1)
    for r in range(world):
        ds = lay.donors_of(r)
        assert r not in ds and len(ds) == world - 1
        assert [lay.peer_index(r, d) for d in ds] == list(range(1, world))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_split_roles(world):
    lay = DonorLayout.split_roles(world, 64)
    assert set(lay.compute).isdisjoint(lay.donors)
    assert sorted(lay.compute + lay.donors) == list(range(world))
    for d in lay.donors:
        assert lay.readers_of(d) == list(lay.compute)
        assert lay.slab_bytes(d) == 64 * len(lay.compute)
    with pytest.raises(ValueError):
        lay.section(lay.compute[0], lay.donors[0])  # a donor-only rank reads nobody
    with pytest.raises(ValueError):
        DonorLayout.split_roles(1, 64)


@pytest.mark.parametrize("n", [1, 3, 7])
def test_preferred_peer_is_a_permutation_over_ranks(n):
    for k in range(25):
        layer, e = divmod(k, 5)
        prefs = [preferred_peer(layer, e, 5, r, n) for r in range(n)]
        assert sorted(prefs) == list(range(1, n + 1))


def test_per_reader_bytes():
    assert per_reader_bytes(1440, 17_301_504, 7) == 206 * 17_301_504
    assert per_reader_bytes(10, 4, 3, extra=5) == 4 * 4 + 5
    with pytest.raises(ValueError):
        per_reader_bytes(1, 1, 0)


# ---- the multi-process path (gloo)

def _rank_main(rank, world, port, q, split):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_00328_b200.cluster import RankGroup, place_experts
        from paper_2602_00328_b200.moe import ExpertResidency
        from paper_2602_00328_b200.memalloc import Tier
        from paper_2602_00328_b200.runtime import virtual_runtime
        from paper_2602_00328_b200.system import build_topology
        g = RankGroup(world, rank)
        m = MODEL
        n_donors = world // 2 if split else world - 1
        lay = (DonorLayout.split_roles if split else DonorLayout.symmetric)(
            world, per_reader_bytes(m.num_layers * m.num_experts, m.expert_size, n_donors))
        # stand-in for PeerPool.export_ipc(): what the slab owner publishes
        handles = g.all_gather({"donor": rank, "slab_bytes": lay.slab_bytes(rank)} if rank in lay.donors else None)
        allocs = []
        if rank in lay.compute:
            donors = lay.donors_of(rank)
            for d in donors:
                assert handles[d] == {"donor": d, "slab_bytes": lay.slab_bytes(d)}
            topo = build_topology(len(donors), [lay.section(d, rank)[1] for d in donors], host_capacity=1 << 40)
            rt = virtual_runtime(topo)
            res = ExpertResidency(m)
            placed, seeds = place_experts(rt, m, res, rank, len(donors))
            assert len(placed) == m.num_layers * m.num_experts
            assert all(res.get(l, e).tier == Tier.PEER_HBM for l in range(m.num_layers)
                       for e in range(m.num_experts))
            for k, h in enumerate(placed):
                d = donors[h.device_id - 1]
                off, size = lay.section(d, rank)
                assert 0 <= h.base and h.base + h.size <= size
                allocs.append((k, d, off + h.base, off + h.base + h.size))
        everything = g.all_gather(allocs)
        # rank group plumbing: max over ranks, rank-0 decisions, any()
        assert g.max(float(rank)) == world - 1
        assert g.min(float(rank)) == 0
        assert g.decide(["ldg", rank]) == ["ldg", 0]
        assert g.any(rank == world - 1) and not g.any(False)
        g.barrier()
        if rank == 0:
            q.put(("ok", everything, lay))
    except BaseException as e:  # surface the failure to the parent
        q.put(("error", rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,split", [(2, False), (4, False), (4, True)])
def test_multi_rank_placement_gloo(world, split):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q, split)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    errs = [m for m in msgs if m[0] == "error"]
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    (_, everything, lay), = [m for m in msgs if m[0] == "ok"]
    m = MODEL
    n_obj = m.num_layers * m.num_experts
    per_donor = {d: [] for d in lay.donors}
    for rank, allocs in enumerate(everything):
        if rank not in lay.compute:
            assert allocs == []
            continue
        assert len(allocs) == n_obj
        for k, d, b0, b1 in allocs:
            assert d != rank and 0 <= b0 < b1 <= lay.slab_bytes(d)
            per_donor[d].append((b0, b1))
        # every reader spreads its experts evenly over its donors
        counts = [sum(1 for a in allocs if a[1] == d) for d in lay.donors_of(rank)]
        assert max(counts) - min(counts) <= 1, counts
    for d, iv in per_donor.items():
        assert not _overlaps(iv), f"readers overlap inside donor {d}'s slab"
    # lockstep readers: at one expert index, the symmetric layout's readers
    # land on distinct donors whenever there are as many donors as readers
    if not lay.compute or split:
        return
    for k in range(n_obj):
        on = [dict((a[0], a[1]) for a in everything[r])[k] for r in lay.compute]
        assert len(set(on)) == len(on)


# ---- NodePools: collective fallback and teardown (no GPU here)

def _nodepools_main(rank, world, port, q, split):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_00328_b200.cluster import RankGroup
        from paper_2602_00328_b200.pool import NodePools
        g = RankGroup(world, rank)
        lay = (DonorLayout.split_roles if split else DonorLayout.symmetric)(world, 64 << 20)
        node = NodePools(g, lay, rank, lambda r: r, mode="remote", tag="cpu-test")
        # no CUDA device: the remote setup fails somewhere, so EVERY rank falls
        # back to ipc together (collective decision), which fails too; the
        # error is recorded, no rank hangs, and close() stays collective
        out = (node.mode, node.error is not None, len(node.views))
        node.close()
        g.barrier()
        q.put(("ok", rank, out))
    except BaseException as e:  # surface the failure to the parent
        q.put(("error", rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,split", [(2, False), (4, True)])
def test_nodepools_fall_back_together_and_close(world, split):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nodepools_main, args=(r, world, port, q, split)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert not [m for m in msgs if m[0] == "error"], msgs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    outs = {m[1]: m[2] for m in msgs}
    assert len(outs) == world
    assert all(o[0] == "ipc" for o in outs.values())          # one decision for all ranks
    assert all(o[2] == 0 for o in outs.values())              # and no half-built views


def test_donation_socket_framing_passes_file_descriptors():
    """The DonorServer / RemotePool wire format: length-prefixed JSON, with
    the chunk's file descriptor riding on the reply (SCM_RIGHTS)."""
    import socket as S
    from paper_2602_00328_b200.pool import _recv_msg, _send_msg
    a, b = S.socketpair(S.AF_UNIX, S.SOCK_STREAM)
    r, w = os.pipe()
    try:
        _send_msg(a, {"op": "create", "chunk": 7})
        assert _recv_msg(b) == {"op": "create", "chunk": 7}
        _send_msg(b, {"ok": True, "bytes": 1 << 25}, fds=[w])
        msg, fds = _recv_msg(a, want_fds=True)
        assert msg == {"ok": True, "bytes": 1 << 25} and len(fds) == 1
        os.write(fds[0], b"chunk")                             # the received fd is the pipe's write end
        assert os.read(r, 5) == b"chunk"
        os.close(fds[0])
    finally:
        for fd in (r, w):
            os.close(fd)
        a.close()
        b.close()
