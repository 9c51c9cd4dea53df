"""The C-ABI library loads without a GPU, exports every symbol declared in
include/harvest_b200.h, and its native allocator makes the reference's exact
decisions (tests/golden/allocator.json, memalloc.py:90-138)."""
import ctypes as C
import json
import os
import random
import re

import pytest

from paper_2602_00328_b200 import _native as N
from paper_2602_00328_b200 import memalloc as M
from oracle import harvest_oracle as O

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(REPO, "include", "harvest_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(hv_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = N.load()
    syms = header_symbols()
    assert len(syms) >= 50
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(N.exported_symbols())
    assert lib.hv_abi_version() == 1


def test_error_strings_and_no_device_behaviour():
    lib = N.load()
    assert lib.hv_error_string(0) == b"ok"
    assert lib.hv_error_string(-2) == b"no capacity"
    n = C.c_int(-1)
    assert lib.hv_device_count(C.byref(n)) == 0
    assert n.value >= 0


def test_native_allocator_matches_reference_runs():
    g = json.load(open(os.path.join(REPO, "tests", "golden", "allocator.json")))
    for case in g["cases"]:
        st = M.init_device(M.DeviceSpec(1, M.Tier.PEER_HBM, case["usable"]))
        for kind, a, b, want in case["ops"]:
            if kind == "alloc":
                seg = M.alloc_best_fit(st, a)
                assert (None if seg is None else seg.base) == want
            else:
                M.free_segment(st, M.Segment(a, b))
            M.check_invariants(st)
        assert [[s.base, s.size] for s in st.free_list] == case["free_list"]
        assert M.allocated_bytes(st) == case["allocated_bytes"]


def test_native_allocator_vs_oracle_random():
    rng = random.Random(3)
    for trial in range(20):
        usable = rng.choice([1000, 1 << 30])
        st = M.init_device(M.DeviceSpec(1, M.Tier.PEER_HBM, usable))
        fl, live = [(0, usable)], []
        for _ in range(300):
            if live and rng.random() < 0.4:
                base, size = live.pop(rng.randrange(len(live)))
                M.free_segment(st, M.Segment(base, size))
                fl = O.free_coalesce(fl, base, size)
            else:
                size = rng.randint(1, usable // rng.choice([5, 40, 300]))
                seg = M.alloc_best_fit(st, size)
                want, fl = O.best_fit(fl, size)
                assert (None if seg is None else seg.base) == want
                if seg is not None:
                    live.append((seg.base, size))
            assert [(s.base, s.size) for s in st.free_list] == fl


def test_allocator_errors_spec():
    # SPEC.md:47-49, 64-67
    st = M.init_device(M.DeviceSpec(1, M.Tier.PEER_HBM, 100, reserved=20))
    assert [(s.base, s.size) for s in st.free_list] == [(0, 80)]
    with pytest.raises(ValueError):
        M.init_device(M.DeviceSpec(1, M.Tier.PEER_HBM, 10, reserved=8, headroom=4))
    with pytest.raises(M.DoubleFreeError):
        M.free_segment(st, M.Segment(5, 3))
    a = M.alloc_best_fit(st, 10)
    b = M.alloc_best_fit(st, 10)
    M.free_segment(st, a)
    M.free_segment(st, b)
    assert [(s.base, s.size) for s in st.free_list] == [(0, 80)]
    with pytest.raises(M.DoubleFreeError):
        M.free_segment(st, a)
    with pytest.raises(ValueError):
        M.alloc_best_fit(st, 0)
    assert M.alloc_best_fit(st, 81) is None


def test_launch_entry_points_validate_arguments_without_a_gpu():
    """Argument errors are reported as HV_E_INVALID before any device work,
    and empty batches are no-ops (so both hold on a CPU-only host)."""
    lib = N.load()
    INV = N.HV_E_INVALID
    page = 65536
    # K1 pointer form: pages but no source / no destination
    assert lib.hv_kv_gather(0, 0, 0, 5, page, 0, 0, None) == INV
    assert lib.hv_kv_gather(0x1000, 0, 0, 5, page, 0, 0, None) == INV
    assert lib.hv_kv_gather(0, 0, 0, 0, page, 0, 0, None) == N.HV_OK
    assert lib.hv_kv_gather(0x1000, 0, 0x2000, (1 << 30) + 1, page, 0, 0, None) == INV
    # K1 table and block-table forms
    assert lib.hv_kv_gather_table(0, 0x1000, 0x2000, 0, 3, page, 0, 0, None) == INV
    assert lib.hv_kv_gather_table(0, 0, 0, 0, 0, page, 0, 0, None) == N.HV_OK
    assert lib.hv_kv_gather_blocks(0x1000, 0x1000, 0, 0x1000, 4, 32, page, 0, 0, None) == INV
    assert lib.hv_kv_gather_blocks(0, 0, 0, 0, 0, 32, page, 0, 0, None) == N.HV_OK
    assert lib.hv_kv_gather_blocks(0x1000, 0x1000, 0x1000, 0x1000, 4, 0, page, 0, 0, None) == N.HV_OK
    # K2 and the host-array forms
    assert lib.hv_batch_copy(0, 0x1000, 0x1000, 2, 0, 0, None) == INV
    assert lib.hv_batch_copy(0, 0, 0, 0, 0, 0, None) == N.HV_OK
    assert lib.hv_swap_blocks_batch(None, None, None, 3, 0, 0, None) == INV
    assert lib.hv_ce_batch_copy(None, None, None, 3, 1, None) == INV
    # content kernels
    assert lib.hv_fill_content(0, 0x1000, 0x1000, 1, None) == INV
    assert lib.hv_digest(0x1000, 0x1000, 1, 0, None) == INV
    assert lib.hv_verify_content(0x1000, 0x1000, 0x1000, 1, 0, None) == INV
    # fused expert FFN: empty launches are no-ops; bad shapes / missing tables are rejected
    A = 0x1000
    assert lib.hv_expert_ffn_gate_up(A, A, A, A, A, A, 0, 2048, 1408, None) == N.HV_OK
    assert lib.hv_expert_ffn_gate_up(A, A, A, 0, A, A, 4, 2048, 1408, None) == INV      # no pair -> row map
    assert lib.hv_expert_ffn_gate_up(A, A, A, A, A, A, 4, 2048, 1400, None) == INV      # I % 64
    assert lib.hv_expert_ffn_down(A, A, A, A, A, 4, 2000, 1408, None) == INV            # H % 64
    assert lib.hv_expert_ffn_down(0, A, A, A, A, 4, 2048, 1408, None) == INV            # no address table
    assert lib.hv_expert_ffn_down(A, A, A, A, A, 70000, 2048, 1408, None) == INV        # grid.y limit
    assert N.c_int_out("hv_expert_ffn_max_tokens") == 64
    # paged decode attention: empty batch is a no-op; unsupported shapes are rejected
    def attn(batch=2, qh=32, kvh=8, d=128, bt=16, splits=4, ptr=A):
        return lib.hv_paged_decode_attention(ptr, A, A, A, A, A, batch, qh, kvh, d, bt, splits, 0.1, None)
    assert attn(batch=0) == N.HV_OK
    assert attn(ptr=0) == INV                # no page table
    assert attn(qh=30) == INV                # q heads not a multiple of KV heads
    assert attn(qh=8 * 16) == INV            # group of 16 query heads per KV head
    assert attn(d=96) == INV                 # head_dim 64 or 128 only
    assert attn(bt=32) == INV                # 16-token blocks
    assert attn(splits=0) == INV
    # K5 flags: balanced (stream-K) form needs batch <= 256; unknown flags are rejected
    def attn_ex(batch=2, flags=N.ATTN_BALANCED):
        return lib.hv_paged_decode_attention_ex(A, A, A, A, A, A, batch, 32, 8, 128, 16, 148, 0.1, flags, None)
    assert attn_ex(batch=257) == INV
    assert attn_ex(flags=8) == INV
    # tiled K4: rows must be multiples of 128 (the tcgen05 kernel); unknown flags rejected
    assert lib.hv_expert_ffn_gate_up_ex(A, A, A, A, A, A, 4, 2048, 1408, 16, None) == INV
    assert lib.hv_expert_ffn_down_ex(A, A, A, A, A, 4, 2048, 1408, 16, None) == INV
    # decode glue: empty batches are no-ops; limits of the route kernel are enforced
    def route(T=32, H=2048, E=60, k=4, ptr=A, flags=0):
        return lib.hv_moe_route(ptr, A, T, H, E, k, A, A, A, A, A, A, A, A, flags, None)
    assert route(T=0) == N.HV_OK
    assert route(ptr=0) == INV
    assert route(E=257) == INV
    assert route(k=9) == INV
    assert route(T=257) == INV
    assert route(H=2047) == INV
    assert route(flags=2) == INV
    assert lib.hv_moe_combine(A, A, A, A, 0, 2048, 4, 1.0, 0, None) == N.HV_OK
    assert lib.hv_moe_combine(A, A, A, A, 4, 2048, 9, 1.0, 0, None) == INV
    assert lib.hv_moe_stage_plan(A, A, A, 1 << 32, 0, 60, A, A, A, None) == INV      # zero slot size
    assert lib.hv_moe_stage_plan(A, A, A, 1 << 32, 4096, 0, A, A, A, None) == N.HV_OK
    # the Python layer raises the matching exception type
    with pytest.raises(N.HarvestNativeError) as ei:
        N.call("hv_batch_copy", 0, 0x1000, 0x1000, 2, 0, 0, None)
    assert ei.value.status == INV


def test_fetch_wrappers_reject_bad_tensors_without_a_gpu():
    import torch
    from paper_2602_00328_b200 import fetch as F
    cpu = torch.zeros(4, dtype=torch.int64)
    with pytest.raises(ValueError, match="CUDA"):
        F.kv_gather(cpu, 65536, dst_page_ptrs=cpu)
    with pytest.raises(ValueError, match="need dst"):
        F.kv_gather(cpu, 65536)
    with pytest.raises(ValueError, match="equal length"):
        F.kv_gather_blocks(cpu, cpu[:3], cpu, cpu, 32, 65536)
    with pytest.raises(ValueError, match="equal length"):
        F.batch_copy(cpu, cpu[:2], cpu)
    with pytest.raises(ValueError, match="length mismatch"):
        F.swap_blocks_batch([1, 2], [3], [4, 5])


def _placer(kind, budget=float("inf"), burst=float("nan"), window=10.0, maxrev=3):
    h = C.c_void_p()
    N.call("hv_placer_create", kind, budget, burst, window, maxrev, C.byref(h))
    return h


def test_native_placer_matches_oracle_selection_random():
    """hv_placer_select / hv_placer_alloc against the oracle's restatement of
    select_peer (runtime.py:155-196) on random donor states, BestFit and
    Locality, random ceilings and candidate subsets."""
    lib = N.load()
    rng = random.Random(11)
    for trial in range(60):
        kind = rng.choice([0, 1])
        p = _placer(kind)
        states, cands, hops = {}, [], {}
        for dev in rng.sample(range(1, 12), rng.randint(1, 6)):
            st = M.init_device(M.DeviceSpec(dev, M.Tier.PEER_HBM, rng.randint(1, 64) << 20))
            for _ in range(rng.randint(0, 12)):
                seg = M.alloc_best_fit(st, rng.randint(1, 8) << 18)
                if seg is not None and rng.random() < 0.4:
                    M.free_segment(st, seg)
            ceiling = rng.choice([st.spec.usable, rng.randint(0, st.spec.usable)])
            hops[dev] = rng.randint(1, 3)
            N.call("hv_placer_add_donor", p, dev, st._h, ceiling, hops[dev])
            states[dev] = st
            cands.append(dict(dev=dev, free_list=[(s.base, s.size) for s in st.free_list],
                              allocated=M.allocated_bytes(st), ceiling=ceiling))
        for _ in range(8):
            size = rng.randint(1, 16) << 18
            sub = [c for c in cands if rng.random() < 0.7]
            want = O.select_device(sub, size, "Locality" if kind == 1 else "BestFit", hops) if sub else None
            ids = (C.c_int * max(1, len(sub)))(*[c["dev"] for c in sub])
            dev = C.c_int(-2)
            st = lib.hv_placer_select(p, size, 0, 0.0, ids, len(sub), C.byref(dev))
            assert (None if st == N.HV_E_NOCAPACITY else dev.value) == want
        lib.hv_placer_destroy(p)


def test_native_placer_token_bucket_and_revocation_window():
    """runtime.py:237-265: a client's bucket starts full at the burst, refills
    at the budget rate up to the burst; the Stability window drops
    revocations older than the window."""
    lib = N.load()
    p = _placer(2, budget=100.0, burst=1000.0)
    tok = C.c_double()
    N.call("hv_placer_tokens", p, 0, 0.0, C.byref(tok))
    assert tok.value == 1000.0
    N.call("hv_placer_spend", p, 0, 900, 0.0)
    N.call("hv_placer_tokens", p, 0, 2.0, C.byref(tok))
    assert tok.value == 300.0
    N.call("hv_placer_tokens", p, 0, 50.0, C.byref(tok))
    assert tok.value == 1000.0
    N.call("hv_placer_tokens", p, 7, 50.0, C.byref(tok))   # another client: its own full bucket
    assert tok.value == 1000.0
    lib.hv_placer_destroy(p)
    p = _placer(3, window=2.0, maxrev=2)
    st = M.init_device(M.DeviceSpec(4, M.Tier.PEER_HBM, 1 << 20))
    N.call("hv_placer_add_donor", p, 4, st._h, 1 << 20, 1)
    for t in (0.0, 1.0, 1.5):
        N.call("hv_placer_note_revocation", p, 4, t)
    n = C.c_int64()
    N.call("hv_placer_churn", p, 4, 2.5, C.byref(n))
    assert n.value == 2                                    # t=0.0 is older than 2.5 - 2.0
    ids, dev = (C.c_int * 1)(4), C.c_int()
    assert lib.hv_placer_select(p, 1024, 0, 2.5, ids, 1, C.byref(dev)) == N.HV_E_NOCAPACITY
    assert lib.hv_placer_select(p, 1024, 0, 3.1, ids, 1, C.byref(dev)) == N.HV_OK and dev.value == 4
    base = C.c_uint64()
    assert lib.hv_placer_alloc(p, 1 << 20, 0, 3.1, None, 0, C.byref(dev), C.byref(base)) == N.HV_OK
    assert (dev.value, base.value, M.allocated_bytes(st)) == (4, 0, 1 << 20)
    assert lib.hv_placer_alloc(p, 1, 0, 3.1, None, 0, C.byref(dev), C.byref(base)) == N.HV_E_NOCAPACITY
    lib.hv_placer_destroy(p)
