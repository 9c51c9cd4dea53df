"""Config 5 on one GPU: a donor availability timeline revokes peer experts in
the middle of a decode and gives capacity back later; rebalance re-places the
experts.  Decode outputs must stay bit-identical to an all-local run and the
release ordering must hold on the real event log (verify.py:25-69)."""
import time

import numpy as np
import pytest
import torch

from tests import refcheck
from tests.test_gpu_decode import RS, _all_local, _tiny

pytestmark = pytest.mark.gpu


def test_donor_monitor_reclaims_under_cotenant_pressure():
    """Co-tenant pressure on the donor (simulated free-memory readings on top
    of a real cudaMemGetInfo probe) revokes LRU handles in order and returns
    their VMM chunks to the donor."""
    from paper_2602_00328_b200.churn import DonorMonitor, mem_get_info
    from paper_2602_00328_b200.runtime import AllocationHints
    from paper_2602_00328_b200.system import HarvestSystem
    free0, total0 = mem_get_info(0)
    assert 0 < free0 <= total0
    seg = 64 << 20
    sysm = HarvestSystem(0, donors=[0], donor_bytes=16 * seg, host_bytes=1, local_bytes=1)
    rt = sysm.runtime
    hs = [rt.harvest_alloc(seg, AllocationHints(client_id="t")) for _ in range(10)]
    assert all(h is not None for h in hs) and sysm.pools[1].committed_bytes == 10 * seg
    fired = []
    for h in hs:
        rt.harvest_register_cb(h, lambda hh, r: fired.append(hh.generation))
    for h in hs[5:]:
        rt.touch(h)          # make hs[0..4] the least recently used
    state = {"free": 8 << 30}
    mon = DonorMonitor(sysm, headroom=512 << 20, meminfo=lambda dev: (state["free"], total0))
    mon.poll()
    assert not fired       # plenty of room: nothing happens
    state["free"] = 128 << 20   # a co-tenant took the rest: level = 128M + 640M - 512M = 256M
    mon.poll()
    sysm.loop.run()
    assert sorted(fired) == sorted(h.generation for h in hs[:6])   # LRU first, >= 384 MiB reclaimed
    assert sysm.pools[1].committed_bytes == 4 * seg                 # chunks unmapped back to the donor
    assert refcheck.verify_release_ordering(sysm.loop.log) == []
    sysm.close()


def test_decode_under_churn_matches_all_local():
    from paper_2602_00328_b200.churn import expert_tier_counts
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore, rebalance
    from paper_2602_00328_b200.system import HarvestSystem
    model = _tiny()
    L, E, S = model.num_layers, model.num_experts, model.expert_size
    cap = 12 * S
    sysm = HarvestSystem(0, donors=[0], donor_bytes=cap, host_bytes=L * E * S, local_bytes=1 << 20)
    store = ExpertStore(model, sysm.host_id, sysm.host)
    store.fill_host(0, weights=True)
    res = ExpertResidency(model)
    counts = np.arange(L * E, dtype=np.int64).reshape(L, E)[::-1].copy()
    replace = lambda: rebalance(sysm.loop, sysm.runtime, model, res, counts, sysm.host_id, store=store)
    replace()
    sysm.loop.run()
    assert expert_tier_counts(res)["PeerHBM"] == 12
    fetcher = ExpertFetcher(sysm.runtime, model, res, store)
    dec = MoEDecoder(fetcher, tokens=16, microbatches=2, seed=0, residual_scale=RS)
    # availability steps at chosen decode steps: full -> 1/3 -> 0 -> full
    levels = {1: cap // 3, 2: 0, 4: cap}
    h = dec.x0
    peer_counts = []
    steps = 7
    for k in range(steps):
        if k in levels:
            sysm.runtime.set_availability(1, levels[k])   # runtime.py:476-487
        h = dec.step(h)          # reads of handles revoked meanwhile extend their drain
        sysm.loop.run()          # drain -> invalidate -> callback -> free
        replace()                # re-place on whatever capacity is left
        sysm.loop.run()
        peer_counts.append(expert_tier_counts(res)["PeerHBM"])
    torch.cuda.synchronize()
    revokes = sysm.loop.log.of_kind("revoke_begin")
    assert revokes and all(r.data["reason"] == "ExternalReclaim" for r in revokes)
    assert peer_counts[1] <= 4 and peer_counts[2] == 0 and peer_counts[3] == 0   # fell back to host
    assert peer_counts[-1] == 12                                                   # re-placed
    assert refcheck.verify_release_ordering(sysm.loop.log) == []
    sys2, dec2, _keep = _all_local(model, 16, 2, 0, store)
    h2 = dec2.x0
    for _ in range(steps):
        h2 = dec2.step(h2)
    torch.cuda.synchronize()
    assert torch.equal(h.view(torch.int16), h2.view(torch.int16))
    sysm.close()
    sys2.close()


def test_markov_churn_wall_clock():
    """ChurnDriver on a wall-clock Markov timeline (traces.py:190-213 with
    50 ms sojourns): whatever the interleaving with decode steps, outputs
    equal the all-local run and the ordering invariants hold."""
    from paper_2602_00328_b200.churn import ChurnDriver, markov_availability
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore, rebalance
    from paper_2602_00328_b200.system import HarvestSystem
    model = _tiny()
    L, E, S = model.num_layers, model.num_experts, model.expert_size
    cap = 12 * S
    sysm = HarvestSystem(0, donors=[0], donor_bytes=cap, host_bytes=L * E * S, local_bytes=1 << 20)
    store = ExpertStore(model, sysm.host_id, sysm.host)
    store.fill_host(0, weights=True)
    res = ExpertResidency(model)
    counts = np.ones((L, E), dtype=np.int64)
    replace = lambda: rebalance(sysm.loop, sysm.runtime, model, res, counts, sysm.host_id, store=store)
    replace()
    sysm.loop.run()
    dec = MoEDecoder(ExpertFetcher(sysm.runtime, model, res, store), tokens=16, microbatches=2, seed=0,
                     residual_scale=RS)
    h = dec.step(dec.x0)                       # warm up before the clock starts
    drv = ChurnDriver(sysm, {1: markov_availability([0, cap // 2, cap], [0.05] * 3, seed=5, horizon=0.6)})
    drv.start()
    steps = 1
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.7:
        h = dec.step(h)
        steps += 1
        drv.tick(replace)
    torch.cuda.synchronize()
    sysm.loop.run()
    assert sysm.loop.log.of_kind("availability_step")
    assert refcheck.verify_release_ordering(sysm.loop.log) == []
    sys2, dec2, _keep = _all_local(model, 16, 2, 0, store)
    h2 = dec2.x0
    for _ in range(steps):
        h2 = dec2.step(h2)
    torch.cuda.synchronize()
    assert torch.equal(h.view(torch.int16), h2.view(torch.int16))
    sysm.close()
    sys2.close()
