"""2-rank NCCL smoke of cluster.RankGroup (handle all_gather, decide, max,
any, barrier) -- the only collectives bench.py issues at N>1.  Launch:
  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29533 tools/nccl_rankgroup_smoke.py [--same-gpu]
--same-gpu puts both ranks on cuda:0 (NCCL normally rejects duplicate GPUs
in one communicator; the script reports what happened either way)."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200.cluster import RankGroup  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = 0 if "--same-gpu" in sys.argv else int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(dev)
out = {"rank": rank, "device": dev}
try:
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
    g = RankGroup(world, rank, device=f"cuda:{dev}")
    hs = g.all_gather(bytes([rank]) * 64)                 # IPC-handle-sized payloads
    assert hs == [bytes([r]) * 64 for r in range(world)]
    assert g.decide(["tma", 296] if rank == 0 else None) == ["tma", 296]
    assert g.max(float(rank) + 0.5) == world - 0.5
    assert g.any(rank == world - 1) and not g.any(False)
    g.barrier()
    out["ok"] = True
    dist.destroy_process_group()
except Exception as e:   # noqa: BLE001
    out["ok"] = False
    out["error"] = repr(e)[:400]
print(json.dumps(out), flush=True)
