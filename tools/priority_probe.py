"""Fetch-stream priority in the staged MoE decode (CUPTI timeline r4c: each
stage's K2 fetch waited ~60 us for the FFN GEMM's CTAs to drain before its
own CTAs were dispatched).  Qwen 8-layer slice, every expert in a self-donor
VMM pool (HBM "peer"), staged decode with 2 micro-batches: ms per step with
the fetch stream at the least / greatest priority, eager and as a CUDA graph
(torch's instantiation, or the library's with per-node priority).  Outputs
must be bit-identical across variants.  Prints JSON."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from benchlib.workload import QWEN15  # noqa: E402
from paper_2602_00328_b200 import _native as N  # noqa: E402
from paper_2602_00328_b200.decode import MoEDecoder  # noqa: E402
from paper_2602_00328_b200.memalloc import Tier  # noqa: E402
from paper_2602_00328_b200.moe import (ExpertFetcher, ExpertResidency, ExpertStore, MoEProfile,  # noqa: E402
                                       RoutingTrace, place_offloaded)
from paper_2602_00328_b200.system import HarvestSystem  # noqa: E402
import ctypes as C  # noqa: E402


def timed(fn, steps=6):
    for _ in range(2):
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
    lo, hi = C.c_int(), C.c_int()
    N.call("hv_stream_priority_range", 0, C.byref(lo), C.byref(hi))
    m = MoEProfile(QWEN15.name, 8, QWEN15.num_experts, QWEN15.top_k, QWEN15.expert_size, hidden=QWEN15.hidden,
                   intermediate=QWEN15.intermediate)
    nbytes = m.num_layers * m.num_experts * m.expert_size
    res = {"priority_range": {"least": lo.value, "greatest": hi.value}}
    ref = None
    for prio in (lo.value, hi.value):
        os.environ["HV_FETCH_PRIORITY"] = str(prio)
        sysm = HarvestSystem(0, donors=[0], donor_bytes=nbytes + (64 << 20), host_bytes=nbytes, local_bytes=1,
                             log_transfers=False)
        store = ExpertStore(m, sysm.host_id, sysm.host)
        store.fill_host(0, weights=True)
        residency = ExpertResidency(m)
        trace = RoutingTrace(1, m.num_layers, m.num_experts, [], np.ones((m.num_layers, m.num_experts), np.int64))
        place_offloaded(sysm.loop, sysm.runtime, m, residency, trace, 100, Tier.PEER_HBM, sysm.host_id, store=store)
        sysm.loop.run()
        f = ExpertFetcher(sysm.runtime, m, residency, store)
        for ctas in (64, 0):
            for mode in ("eager", "graph", "graph_node_priority"):
                dec = MoEDecoder(f, tokens=32, microbatches=2, seed=0, max_ctas=ctas)
                if mode != "eager":
                    dec.capture_graph(node_priority=(mode == "graph_node_priority"))
                out, ms = timed(lambda: dec.step(dec.x0))
                if ref is None:
                    ref = out
                key = f"prio{prio}_ctas{ctas}_{mode}"
                res[key] = {"ms_per_step": ms, "tokens_per_s": 32 / (ms * 1e-3),
                            "bit_identical": bool(torch.equal(out, ref))}
                print(key, json.dumps(res[key]), flush=True)
                del dec
                torch.cuda.synchronize()
                sysm.loop.run()
        sysm.close()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
