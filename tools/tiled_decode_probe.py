"""MoE decode with the experts stored row-major vs as HV_FFN_TILED tiles
(the tcgen05 K4 streams each 16 KiB weight tile as one bulk copy).  Qwen
8-layer slice, batch 32, every expert in a self-donor VMM pool (the HBM
"peer" stand-in) or all local; fused (K4 in place) and staged (K2 into the
staging slots, then the FFN: cuBLAS bmm over row-major experts, K4 over tiled
ones), one micro-batch, each step a CUDA graph.  Tiled outputs must equal the
row-major fused outputs bit for bit (K4 reads the same logical weights).
Prints JSON: ms per step and tokens/s."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from benchlib.workload import QWEN15  # noqa: E402
from paper_2602_00328_b200.decode import MoEDecoder  # noqa: E402
from paper_2602_00328_b200.memalloc import Tier  # noqa: E402
from paper_2602_00328_b200.moe import (ExpertFetcher, ExpertResidency, ExpertStore, MoEProfile,  # noqa: E402
                                       RoutingTrace, place_offloaded)
from paper_2602_00328_b200.system import HarvestSystem  # noqa: E402


def timed(fn, steps=8):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        out = fn()
    e1.record()
    e1.synchronize()
    return out.clone(), e0.elapsed_time(e1) / steps


def main():
    layers = int(os.environ.get("HV_PROBE_LAYERS", "8"))
    m = MoEProfile(QWEN15.name, layers, QWEN15.num_experts, QWEN15.top_k, QWEN15.expert_size, hidden=QWEN15.hidden,
                   intermediate=QWEN15.intermediate)
    L, E, S = m.num_layers, m.num_experts, m.expert_size
    nbytes = L * E * S
    res, ref = {"model": f"{m.name} slice: {L} layers x {E} experts x {S} B, batch 32, top-4"}, None
    for layout in ("row", "tiled"):
        sysm = HarvestSystem(0, donors=[0], donor_bytes=nbytes + (64 << 20), host_bytes=nbytes, local_bytes=1,
                             log_transfers=False)
        store = ExpertStore(m, sysm.host_id, sysm.host)
        store.fill_host(0, weights=True, layout=layout)
        residency = ExpertResidency(m)
        trace = RoutingTrace(1, L, E, [], np.ones((L, E), np.int64))
        place_offloaded(sysm.loop, sysm.runtime, m, residency, trace, 100, Tier.PEER_HBM, sysm.host_id, store=store)
        sysm.loop.run()
        f = ExpertFetcher(sysm.runtime, m, residency, store)
        resident = torch.from_numpy(store.host.view()[:nbytes].copy()).cuda()
        lres = ExpertResidency(m)
        for layer in range(L):
            for e in range(E):
                lres.set_tier(layer, e, Tier.LOCAL_HBM)
        lstore = ExpertStore(m, sysm.host_id, None)
        lstore.layout = layout
        lf = ExpertFetcher(sysm.runtime, m, lres, lstore,
                           local_addr=[[resident.data_ptr() + (layer * E + e) * S for e in range(E)]
                                       for layer in range(L)])
        for where, fetcher in (("peer", f), ("local", lf)):
            for fused in (True, False):
                dec = MoEDecoder(fetcher, tokens=32, microbatches=1, seed=0, fused=fused)
                dec.capture_graph()
                out, ms = timed(lambda: dec.step(dec.x0))
                if ref is None:
                    ref = out
                key = f"{layout}_{where}_{'fused' if fused else 'staged'}"
                res[key] = {"ms_per_step": ms, "tokens_per_s": 32 / (ms * 1e-3),
                            "equals_row_major_fused": bool(torch.equal(out, ref))}
                print(key, json.dumps(res[key]), flush=True)
                del dec
                torch.cuda.synchronize()
                sysm.loop.run()
        del resident
        sysm.close()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
