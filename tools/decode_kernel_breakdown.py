"""Where a fused MoE decode step spends its time: the CUPTI activity trace
(torch.profiler / Kineto) of CUDA-graph-replayed steps of the fused decoder
(Qwen 8-layer slice, batch 32, experts resident in HBM, row-major or tiled),
summed per kernel name, plus the step span and the idle gaps between kernels
on the compute stream.  Prints JSON.

    python tools/decode_kernel_breakdown.py [row|tiled]
"""
import collections
import json
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from benchlib.workload import QWEN15  # noqa: E402
from paper_2602_00328_b200.decode import MoEDecoder  # noqa: E402
from paper_2602_00328_b200.memalloc import Tier  # noqa: E402
from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore, MoEProfile  # noqa: E402
from paper_2602_00328_b200.system import HarvestSystem  # noqa: E402


def main():
    layout = sys.argv[1] if len(sys.argv) > 1 else "tiled"
    m = MoEProfile(QWEN15.name, 8, QWEN15.num_experts, QWEN15.top_k, QWEN15.expert_size, hidden=QWEN15.hidden,
                   intermediate=QWEN15.intermediate)
    L, E, S = m.num_layers, m.num_experts, m.expert_size
    sysm = HarvestSystem(0, host_bytes=L * E * S, local_bytes=1, log_transfers=False)
    store = ExpertStore(m, sysm.host_id, sysm.host)
    store.fill_host(0, weights=True, layout=layout)
    resident = torch.from_numpy(store.host.view()[:L * E * S].copy()).cuda()
    res = ExpertResidency(m)
    for layer in range(L):
        for e in range(E):
            res.set_tier(layer, e, Tier.LOCAL_HBM)
    lstore = ExpertStore(m, sysm.host_id, None)
    lstore.layout = layout
    f = ExpertFetcher(sysm.runtime, m, res, lstore,
                      local_addr=[[resident.data_ptr() + (layer * E + e) * S for e in range(E)] for layer in range(L)])
    dec = MoEDecoder(f, tokens=32, microbatches=1, seed=0, fused=True)
    h = dec.decode(2)
    dec.capture_graph()
    for _ in range(3):
        h = dec.step(h)
    torch.cuda.synchronize()
    steps = 5
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            h = dec.step(h)
        torch.cuda.synchronize()
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    per = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        name = e["name"]
        key = name[:100]
        per[key][0] += 1
        per[key][1] += e["dur"]
    span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
    busy = []
    for e in ev:
        s0, s1 = e["ts"], e["ts"] + e["dur"]
        if busy and s0 <= busy[-1][1]:
            busy[-1][1] = max(busy[-1][1], s1)
        else:
            busy.append([s0, s1])
    gaps = [b[0] - a[1] for a, b in zip(busy, busy[1:])]
    out = {"layout": layout, "steps": steps, "layers": L, "span_us_per_step": span / steps,
           "busy_us_per_step": sum(b - a for a, b in busy) / steps,
           "gap_us_per_step": sum(gaps) / steps, "gaps_per_step": len(gaps) / steps,
           "median_gap_us": float(np.median(gaps)) if gaps else 0.0,
           "kernels_per_step": len(ev) / steps,
           "per_kernel_us_per_step": {k: {"launches_per_step": v[0] / steps, "us_per_step": v[1] / steps}
                                      for k, v in sorted(per.items(), key=lambda kv: -kv[1][1])}}
    print(json.dumps(out, indent=1))
    sysm.close()


if __name__ == "__main__":
    main()
