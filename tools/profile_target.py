"""Short, ncu-friendly driver: a few launches of each fetch kernel at the
bench shapes.  Usage: python tools/profile_target.py MODE [engine] [reps]
MODE: host | hbm | kv | blocks | attn | fused | check (the per-fetch digest
check of one Qwen stage) | checked (fetch + check fused, HBM) | peer | peer_kv (both need 2 GPUs: cuda:1 donates
a VMM pool read by cuda:0 over NVLink; tools/ncu_nvlink.sh captures the
nvlrx/nvltx byte counters of those launches)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200 import fetch as F  # noqa: E402
from paper_2602_00328_b200.pool import HostTier  # noqa: E402


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "host"
    eng = sys.argv[2] if len(sys.argv) > 2 else "ldg"
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    dev = "cuda:0"
    if what in ("host", "hbm"):
        S, n = 17_301_504, 53
        if what == "host":
            tier = HostTier(n * S)
            base = tier.device_address()
        else:
            buf = torch.empty(n * S, dtype=torch.uint8, device=dev)
            base = buf.data_ptr()
        dst = torch.empty(n * S, dtype=torch.uint8, device=dev)
        sp = F.ptrs_tensor([base + i * S for i in range(n)], dev)
        dp = F.ptrs_tensor([dst.data_ptr() + i * S for i in range(n)], dev)
        sz = F.ptrs_tensor([S] * n, dev)
        for _ in range(reps):
            F.batch_copy(sp, dp, sz, engine=eng)
    elif what in ("peer", "peer_kv"):   # NVLink: a VMM pool on cuda:1, read by cuda:0
        from paper_2602_00328_b200 import _native as N
        from paper_2602_00328_b200.pool import PeerPool
        if torch.cuda.device_count() < 2:
            raise SystemExit("peer modes need 2 GPUs")
        N.call("hv_enable_peer_access", 0, 1)
        S, n = 17_301_504, 53
        pool = PeerPool(1, n * S, readers=[0])
        pool.commit(0, n * S)
        F.fill_content(F.ptrs_tensor([pool.va + i * S for i in range(n)], "cuda:1"),
                       F.ptrs_tensor([S] * n, "cuda:1"), list(range(n)))
        torch.cuda.synchronize(1)
        if what == "peer":
            dst = torch.empty(n * S, dtype=torch.uint8, device=dev)
            sp = F.ptrs_tensor([pool.va + i * S for i in range(n)], dev)
            dp = F.ptrs_tensor([dst.data_ptr() + i * S for i in range(n)], dev)
            sz = F.ptrs_tensor([S] * n, dev)
            for _ in range(reps):
                F.batch_copy(sp, dp, sz, engine=eng)
        else:   # config 1's layer: 1,024 x 64 KiB pages at randperm(seed 1) slots of the donor pool
            page, npg = 65536, 1024
            slots = torch.randperm(n * S // page, generator=torch.Generator().manual_seed(1))[:npg]
            src = F.ptrs_tensor([pool.va + int(t) * page for t in slots], dev)
            dst = torch.empty(npg * page, dtype=torch.uint8, device=dev)
            for _ in range(reps):
                F.kv_gather(src, page, dst=dst, engine=eng)
        torch.cuda.synchronize(0)
        pool.decommit(0, n * S)
        pool.close()
    elif what == "checked":   # the fetch with its content check fused (hv_swap_blocks_batch_checked), HBM -> HBM
        from paper_2602_00328_b200 import _native as N
        S, n = 17_301_504, 53
        src = torch.empty(n * S, dtype=torch.uint8, device=dev)
        dst = torch.empty(n * S, dtype=torch.uint8, device=dev)
        sp = np.array([src.data_ptr() + i * S for i in range(n)], dtype=np.uint64)
        dp = np.array([dst.data_ptr() + i * S for i in range(n)], dtype=np.uint64)
        sz = np.full(n, S, dtype=np.uint64)
        exp = np.zeros(n, dtype=np.uint64)
        scratch = torch.zeros(n, dtype=torch.int64, device=dev)
        err = torch.zeros(1, dtype=torch.int64, device=dev)
        for _ in range(reps):
            N.call("hv_swap_blocks_batch_checked", sp.ctypes.data, dp.ctypes.data, sz.ctypes.data, exp.ctypes.data, n,
                   N.ENGINES[eng], 0, scratch.data_ptr(), 0, err.data_ptr(), 0)
    elif what == "check":   # per-fetch content check (hv_check_digests) of one Qwen stage in HBM
        from paper_2602_00328_b200 import _native as N
        S, n = 17_301_504, 53
        buf = torch.empty(n * S, dtype=torch.uint8, device=dev)
        ptrs = np.array([buf.data_ptr() + i * S for i in range(n)], dtype=np.uint64)
        sz = np.full(n, S, dtype=np.uint64)
        exp = np.zeros(n, dtype=np.uint64)
        scratch = torch.zeros(n, dtype=torch.int64, device=dev)
        err = torch.zeros(1, dtype=torch.int64, device=dev)
        for _ in range(reps):
            N.call("hv_check_digests_batch", ptrs.ctypes.data, sz.ctypes.data, exp.ctypes.data, n,
                   scratch.data_ptr(), 0, err.data_ptr(), 0)
    elif what == "blocks":  # KV reload slice: 256 blocks x 32 layers x 64 KiB, [layer][slot] slabs -> cache
        page, L, nb, slab = 65536, 32, 256, 64
        slabs = [torch.empty(L * slab * page, dtype=torch.uint8, device=dev) for _ in range(nb // slab)]
        cache = torch.empty(L * nb * page, dtype=torch.uint8, device=dev)
        order = np.random.default_rng(0).permutation(nb)
        sb = F.ptrs_tensor([slabs[o // slab].data_ptr() + (o % slab) * page for o in order], dev)
        ss = F.ptrs_tensor([slab * page] * nb, dev)
        db = F.ptrs_tensor([cache.data_ptr() + i * page for i in range(nb)], dev)
        ds = F.ptrs_tensor([nb * page] * nb, dev)
        for _ in range(reps):
            F.kv_gather_blocks(sb, ss, db, ds, L, page, engine=eng)
    elif what == "attn":  # K5 paged decode attention, 1 x 128k Llama-3-8B context, pages scattered in HBM
        from paper_2602_00328_b200 import _native as N
        B, ctx, kvh, g, D = 1, 131072, 8, 4, 128
        nb = ctx // 16
        page = 2 * 16 * kvh * D * 2
        pool = torch.empty(nb, page, dtype=torch.uint8, device=dev)
        pool.view(torch.float16).normal_(0, 0.5)
        ptrs = (torch.randperm(nb, device=dev) * page + pool.data_ptr()).to(torch.int64)
        start = torch.tensor([0, nb], dtype=torch.int32, device=dev)
        tok = torch.tensor([ctx], dtype=torch.int32, device=dev)
        q = torch.randn(B, kvh * g, D, device=dev).to(torch.float16)
        out = torch.empty(B, kvh * g, D, device=dev)
        splits = torch.cuda.get_device_properties(0).multi_processor_count // (B * kvh)
        part = torch.empty(B * kvh * splits * g * (D + 2), device=dev)
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(reps):
            N.call("hv_paged_decode_attention", ptrs.data_ptr(), start.data_ptr(), tok.data_ptr(), q.data_ptr(),
                   out.data_ptr(), part.data_ptr(), B, kvh * g, kvh, D, 16, splits, 1 / D ** 0.5, s)
    elif what == "fused":  # fused expert FFN at the Qwen1.5-MoE stage shape, experts in HBM
        from paper_2602_00328_b200 import _native as N
        E, T, k, H, I = 60, 32, 4, 2048, 1408
        S = 3 * H * I * 2
        W = (torch.randn(E * S // 2, device=dev) * 0.02).to(torch.bfloat16)
        h = torch.randn(T, H, device=dev).to(torch.bfloat16)
        topi = torch.randn(T, E, device=dev).topk(k, dim=1).indices.reshape(-1)
        order = torch.argsort(topi, stable=True)
        counts = torch.zeros(E, dtype=torch.int32, device=dev).scatter_add_(0, topi, torch.ones_like(topi, dtype=torch.int32))
        offs = torch.cumsum(counts, 0, dtype=torch.int32) - counts
        tok = torch.div(order, k, rounding_mode="floor").to(torch.int32)
        addr = torch.tensor([W.data_ptr() + e * S for e in range(E)], dtype=torch.int64, device=dev)
        act = torch.empty(T * k, I, dtype=torch.bfloat16, device=dev)
        y = torch.empty(T * k, H, dtype=torch.float32, device=dev)
        s = torch.cuda.current_stream().cuda_stream
        fl = N.FFN_TILED if eng == "tiled" else 0   # the engine argument "tiled": HV_FFN_TILED (random bytes either way)
        for _ in range(reps):
            N.call("hv_expert_ffn_gate_up_ex", addr.data_ptr(), counts.data_ptr(), offs.data_ptr(), tok.data_ptr(),
                   h.data_ptr(), act.data_ptr(), E, H, I, fl, s)
            N.call("hv_expert_ffn_down_ex", addr.data_ptr(), counts.data_ptr(), offs.data_ptr(), act.data_ptr(),
                   y.data_ptr(), E, H, I, fl, s)
        print("active experts", int((counts > 0).sum()))
    else:  # KV config 1: 1024 pages x 64 KiB from 4096 HBM slots
        page, npg, nslots = 65536, 1024, 4096
        slots = torch.empty(nslots * page, dtype=torch.uint8, device=dev)
        perm = np.random.default_rng(1).permutation(nslots)[:npg]
        sp = F.ptrs_tensor([slots.data_ptr() + int(p) * page for p in perm], dev)
        dst = torch.empty(npg * page, dtype=torch.uint8, device=dev)
        for _ in range(reps):
            F.kv_gather(sp, page, dst=dst, engine=eng)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
