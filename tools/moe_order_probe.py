"""Staged MoE decode (K2 fetch on the fetch stream, cuBLAS FFN on the compute
stream), two micro-batches: issue order of stage s+1's fetch against stage s's
FFN, eager and as a CUDA graph (run r115 against a decoder with an
``issue_ahead`` switch that was then dropped: no gain), with the experts in a self-donor VMM pool
(peer tier = this GPU's HBM) or in the pinned host tier.  Qwen1.5-MoE shapes,
8 layers, 32 tokens.  Prints JSON: ms per step; outputs checked equal."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from event_probe import b2b  # noqa: E402
from paper_2602_00328_b200.decode import MoEDecoder  # noqa: E402
from paper_2602_00328_b200.moe import (QWEN15_MOE_A27B, ExpertFetcher, ExpertResidency, ExpertStore,  # noqa: E402
                                       MoEProfile, rebalance)
from paper_2602_00328_b200.system import HarvestSystem  # noqa: E402


def case(tier, layers=8, tokens=32):
    q = QWEN15_MOE_A27B
    model = MoEProfile(q.name, layers, q.num_experts, q.top_k, q.expert_size, hidden=q.hidden,
                       intermediate=q.intermediate)
    L, E, S = layers, q.num_experts, q.expert_size
    sysm = HarvestSystem(0, donors=[0] if tier == "peer" else [], donor_bytes=L * E * S + (64 << 20),
                         host_bytes=L * E * S, local_bytes=1 << 20)
    store = ExpertStore(model, sysm.host_id, sysm.host)
    store.fill_host(0, weights=True)
    res = ExpertResidency(model)
    if tier == "peer":
        rebalance(sysm.loop, sysm.runtime, model, res, np.ones((L, E), dtype=np.int64), sysm.host_id,
                  max_migrations=L * E, store=store)
        sysm.loop.run()
    fetcher = ExpertFetcher(sysm.runtime, model, res, store)
    out, want = {}, None
    for ahead in (False, True):
        for graph in (False, True):
            MoEDecoder.issue_ahead = ahead
            dec = MoEDecoder(fetcher, tokens=tokens, microbatches=2, seed=0)
            if graph:
                dec.capture_graph()
            y = dec.step(dec.x0).clone()
            if want is None:
                want = y
            assert torch.equal(y, want)
            out[f"ahead={int(ahead)} graph={int(graph)}"] = b2b(lambda: dec.step(dec.x0), n=3 if tier == "host" else 10)
            del dec
    MoEDecoder.issue_ahead = True
    return out


if __name__ == "__main__":
    print(json.dumps({"peer_hbm": case("peer"), "host": case("host")}, indent=1))
